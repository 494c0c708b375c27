#!/bin/bash
# Evidence for one K1 revision: bench line (product + fits), ncu launch list,
# one full capture of the product kernel.
# usage (on the GPU box): tools/profile_round.sh TAG [WORKLOAD] [KREGEX]   -> gpurun_out/TAG_*
T=${1:?tag}
W=${2:-cfg3}
K=${3:-"kop_tc_kernel|kop_sym1_kernel|kop_sym2_kernel"}
O=gpurun_out
mkdir -p $O
timeout 1200 python bench.py --workload $W --steps 5 --warmup 3 > $O/${T}_bench.log 2>&1 || { tail $O/${T}_bench.log; exit 1; }
tail -1 $O/${T}_bench.log > $O/${T}_bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${T}_bench_launches.csv python bench.py --workload $W --steps 2 --warmup 1 \
  --no-cpu-baseline --no-fit > $O/${T}_ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 3 -c 1 \
  -o $O/${T}_kop_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-fit \
  > $O/${T}_ncu_full.log 2>&1
ncu -i $O/${T}_kop_$W.ncu-rep --page details > $O/${T}_kop_${W}_details.txt 2>&1
ncu -i $O/${T}_kop_$W.ncu-rep --page raw --csv > $O/${T}_kop_${W}_raw.csv 2>&1
cat $O/${T}_bench_line.json
exit 0
