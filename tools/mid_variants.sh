#!/bin/bash
for v in "$@"; do
  case $v in base) lib=paper_2308_09723_b200/libfq.so;; *) lib=paper_2308_09723_b200/_variants/libfq_$v.so;; esac
  echo "== $v"; FQ_LIB_PATH=$PWD/$lib timeout 300 python tools/mid_m.py 2>&1
done
