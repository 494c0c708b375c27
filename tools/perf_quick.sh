#!/bin/bash
# One GPU call: build, K1 parity tests, K1 timings at n=200k, cfg3 bench line.
make -C paper_2310_20285_b200/csrc -j8 >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_operator.py -x -q 2>&1 | tail -3
timeout 60 python tools/prof_tc.py --n 200000 --family rbf
timeout 60 python tools/prof_tc.py --n 200000 --family matern32
timeout 60 python tools/prof_tc.py --n 200000 --d 50 --w 10
[ "$1" == "bench" ] && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline | tail -1
exit 0
