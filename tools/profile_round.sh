#!/bin/bash
# One GPU call's worth of measurement for a round: the bench line, the
# launch list of the same command, and ncu --set full captures of the K1 /
# K2 / K3 kernels of configs 2, 4 and 5 (tools/profile_step.py).  Every
# profiled command first runs once without ncu.  Outputs in gpurun_out/.
# Usage (on the GPU box): bash tools/profile_round.sh TAG
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
NCU="ncu --clock-control none --import-source on"
python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
    --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/${TAG}_bench_ncu.log 2>&1
echo "launches rc=$?"
# matching launches per step: enclose (+ replay scan for trig fields), three
# rows_kernel passes (+ rows_half_kernel in 3-D/4-D), compaction, K3
declare -A PER=([2]=7 [4]=7 [5]=8)
for c in 2 4 5; do
  python tools/profile_step.py $c > $O/${TAG}_step$c.log 2>&1 || { echo "step $c failed"; continue; }
  # second step: K1 (+ its replay scan), K2 passes, compaction, K3
  $NCU --set full -k regex:'enclose_kernel|rows_kernel|rows_half_kernel|compact_kernel|peel_coop_kernel|enclose_replay' \
      -s ${PER[$c]} -c ${PER[$c]} -o $O/${TAG}_ncu_config$c -f python tools/profile_step.py $c > $O/${TAG}_ncu_config$c.log 2>&1
  echo "ncu config $c rc=$?"
  # condensed here (reports are too large to bring back whole)
  python tools/make_ncu_summary.py $O/${TAG}_ncu_config$c.ncu-rep $O/${TAG}_ncu_config$c.json \
      "ncu --set full -k <K1|K2|K3> python tools/profile_step.py $c (second step)" \
      > $O/${TAG}_ncu_config$c.txt 2>&1
  ncu -i $O/${TAG}_ncu_config$c.ncu-rep --page raw --csv > $O/${TAG}_ncu_config$c.raw.csv 2>/dev/null
  gzip -f $O/${TAG}_ncu_config$c.raw.csv
  rm -f $O/${TAG}_ncu_config$c.ncu-rep
done
du -sh $O
