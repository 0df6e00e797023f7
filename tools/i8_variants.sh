#!/bin/bash
# Diagnostics: time fq_gemm_i8 under libfq build variants (build.build_variant): FQ_I8_DBG
# (1 = no MMA, 2 = no unpack / tcgen05.st), FQ_I8_DG_* (dequant warp groups).
for v in "$@"; do
  case $v in base) lib=paper_2308_09723_b200/libfq.so;; *) lib=paper_2308_09723_b200/_variants/libfq_$v.so;; esac
  echo "== $v"; FQ_LIB_PATH=$PWD/$lib timeout 120 python tools/i8_bench.py --ms ${MS:-1,16,64} 2>&1 | grep -v '^{' | sed 's/, .bf16.*//'
done
