"""C-ABI checks that need no GPU: the library loads, exports every symbol include/longflow.h
declares, and host-side validation returns status codes instead of crashing."""
import ctypes
import re
import os

import pytest

from paper_2603_11504_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "longflow.h")).read()
    return sorted(set(re.findall(r"\b(lf_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    names = _declared()
    for n in ("lf_cache_create", "lf_prefill_fill", "lf_decode_step", "lf_cache_destroy", "lf_cache_bytes"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = binding.load()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(binding.EXPORTS) == _declared()


def test_status_strings():
    lib = binding.load()
    for code, name in binding.STATUS.items():
        assert lib.lf_status_string(code).decode() == name


def test_config_struct_matches_header():
    """binding.CacheConfig mirrors lf_cache_config field by field (names, order, 4-byte types)."""
    src = open(os.path.join(ROOT, "include", "longflow.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} lf_cache_config;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(int32_t|float)\s+(\w+)\s*;", body)
    assert [n for _, n in fields] == [n for n, _ in binding.CacheConfig._fields_]
    assert ctypes.sizeof(binding.CacheConfig) == 4 * len(fields)


@pytest.mark.parametrize("kw,status", [
    (dict(plan_batch=1), 1),              # the global batch smaller than this cache
    (dict(seq_offset=2), 1),              # seq_offset without plan_batch
    (dict(plan_batch=4, seq_offset=3), 1),   # shard past the global batch
    (dict(plan_shards=-1), 1),
    (dict(plan_shards=2, solo=True), 1),  # plan_shards plans have no whole-unit rounds
    (dict(ctas_per_sm=3), 1),
    (dict(budget=1), 1),                  # S:125 budget < 2
    (dict(num_q_heads=6, num_kv_heads=4), 1),
    (dict(head_dim=96), 2),               # not built
    (dict(batch=0), 1),
    (dict(split_tokens=100), 1),
    (dict(num_q_heads=34, num_kv_heads=2), 2),   # G = 17
])
def test_host_validation(kw, status):
    args = dict(batch=2, num_q_heads=8, num_kv_heads=2, head_dim=128, budget=64)
    args.update(kw)
    cfg = binding.make_config(**args)
    n = ctypes.c_size_t()
    st = binding.load().lf_cache_bytes(ctypes.byref(cfg), ctypes.byref(n))
    assert st == status
    assert binding.load().lf_last_error()


def test_cache_bytes_layout():
    cfg = binding.make_config(batch=4, num_q_heads=32, num_kv_heads=8, head_dim=128, budget=4096)
    nbytes = binding.cache_bytes(cfg)
    kv = 4 * 8 * 4096 * 128 * 2
    assert 2 * kv <= nbytes < 2 * kv + (1 << 20)


def test_create_without_gpu_is_a_status_not_a_crash():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = binding.make_config(batch=1, num_q_heads=1, num_kv_heads=1, head_dim=64, budget=8)
    h = ctypes.c_void_p()
    st = binding.load().lf_cache_create(ctypes.byref(cfg), 0, None, 0, ctypes.byref(h))
    assert st in (1, 5) and not h.value


def test_missing_extension_fails_loudly():
    """No CPU fallback: with the CUDA library absent, the product path raises."""
    import subprocess
    import sys
    env = dict(os.environ, LF_LIB="/nonexistent/liblongflow.so")
    r = subprocess.run([sys.executable, "-c", "from paper_2603_11504_b200 import Cache; Cache(1, 4, 1, 128, 256)"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "not built" in r.stderr, r.stderr[-2000:]


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly():
    """Without a CUDA device the C ABI reports an error status; nothing computes on the CPU."""
    from paper_2603_11504_b200 import Cache, LFError
    with pytest.raises((LFError, RuntimeError)):
        Cache(1, 4, 1, 128, 256)
