#!/bin/bash
# Per-kernel launch metrics of the EDT on Bernoulli grids (GPU box):
#   tools/edt_profile.sh "512 0.02 0" "512 0.0001 1" ...   [env knobs pass through]
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum
for c in "$@"; do
  echo "== $c"
  ncu --metrics $M --clock-control none --csv --log-file /tmp/ncu_k.csv python tools/edt_time.py $c > /dev/null 2>&1
  python tools/ncu_kernels.py /tmp/ncu_k.csv
done
