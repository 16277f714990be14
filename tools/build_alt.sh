#!/bin/bash
# Build liblongflow.so from an alternative csrc directory (A/B experiments): tools/build_alt.sh <csrc dir> <out.so> [defines...]
src=$1; out=$2; shift 2
defs=""; for d in "$@"; do defs="$defs -D$d"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I$(dirname $0)/../include $defs -o $out $src/lf_runtime.cu $src/lf_decode_simt.cu $src/lf_decode_tc.cu $src/lf_snapkv.cu $src/lf_diag.cu
