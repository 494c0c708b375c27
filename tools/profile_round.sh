#!/bin/bash
# Evidence for one K1 revision: bench line, ncu launch list, one full capture.
# usage (on the GPU box): tools/profile_round.sh TAG [WORKLOAD]   -> gpurun_out/TAG_*
T=${1:?tag}
W=${2:-cfg3}
O=gpurun_out
mkdir -p $O
make -C paper_2310_20285_b200/csrc -j8 >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --workload $W --steps 3 --warmup 3 > $O/${T}_bench.log 2>&1 || { tail $O/${T}_bench.log; exit 1; }
tail -1 $O/${T}_bench.log > $O/${T}_bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${T}_bench_launches.csv python bench.py --workload $W --steps 2 --warmup 1 --no-cpu-baseline \
  > $O/${T}_ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"kop_tc_kernel|kop_sym1_kernel" -s 3 -c 1 \
  -o $O/${T}_kop_tc_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline \
  > $O/${T}_ncu_full.log 2>&1
ncu -i $O/${T}_kop_tc_$W.ncu-rep --page details > $O/${T}_kop_tc_${W}_details.txt 2>&1
ncu -i $O/${T}_kop_tc_$W.ncu-rep --page raw --csv > $O/${T}_kop_tc_${W}_raw.csv 2>&1
cat $O/${T}_bench_line.json
exit 0
