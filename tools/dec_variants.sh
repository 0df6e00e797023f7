#!/bin/bash
# Diagnostics: decode-kernel sweep under libfq build variants (build.build_variant).
for v in "$@"; do
  case $v in base) lib=paper_2308_09723_b200/libfq.so;; *) lib=paper_2308_09723_b200/_variants/libfq_$v.so;; esac
  echo "== $v"; FQ_LIB_PATH=$PWD/$lib timeout 200 python tools/dec_sweep.py --M ${MS:-1 8 9 16 24 32} 2>&1
done
