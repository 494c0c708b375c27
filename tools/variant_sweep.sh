#!/bin/bash
# Time prebuilt variants of libncgp_b200.so (variants/lib_*.so, built here with
# different -D tuning macros) on the K1 shapes, with the K1 parity tests for each.
for so in variants/lib_*.so; do
  cp "$so" paper_2310_20285_b200/libncgp_b200.so
  echo "== $so"
  timeout 300 python -m pytest tests/test_gpu_operator.py -x -q 2>&1 | tail -1
  timeout 60 python tools/prof_tc.py --n 200000 --family rbf
  timeout 60 python tools/prof_tc.py --n 200000 --family matern32
  timeout 60 python tools/prof_tc.py --n 200000 --d 50 --w 10
done
exit 0
