set -x
timeout 900 python tools/sweep.py --budgets 512,1024,2048,4096,8192 --batches 1,2,4,8,16 --out gpurun_out/sw_lat.jsonl > gpurun_out/sw_lat.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/icache_probe tools/probes/icache_probe.cu && timeout 60 /tmp/icache_probe > gpurun_out/icache_probe.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/lat_probe tools/probes/lat_probe.cu && timeout 60 /tmp/lat_probe > gpurun_out/lat_probe.txt 2>&1
mkdir -p altlib; python -c "from paper_2603_11504_b200.build import build_variant; build_variant('altlib/lib_trace.so', ['LF_TRACE'])" && LF_LIB=altlib/lib_trace.so timeout 120 python tools/trace_run.py q7 > gpurun_out/trace_q7.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_plans.py -q -x > gpurun_out/plans_test.log 2>&1
