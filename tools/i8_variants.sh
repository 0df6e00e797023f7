#!/bin/bash
# Diagnostics: time fq_gemm_i8 with parts of the work removed (FQ_I8_DBG variants of libfq).
for v in base nomma nosttm; do
  case $v in base) lib=paper_2308_09723_b200/libfq.so;; *) lib=paper_2308_09723_b200/_variants/libfq_$v.so;; esac
  echo "== $v"; FQ_LIB_PATH=$PWD/$lib timeout 120 python tools/i8_bench.py --ms 1,16,64 2>&1 | grep -v '^{' | sed 's/, .bf16.*//'
done
