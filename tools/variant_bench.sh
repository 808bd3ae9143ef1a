#!/bin/bash
# Rebuild libvx.so with extra -D flags per variant and report the 512^3 tick
# phases (tuning experiments on the GPU box; the default build is restored last).
#   tools/variant_bench.sh "base:" "w28:-DVX_STREAM_WARPS=28 -DVX_STREAM_CAP=62" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  (cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 EXTRA="$flags" >/dev/null 2>&1) || { echo "$name: build failed"; continue; }
  for rep in 1 2; do
    python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); p=d['phase_ms']
print('$name', 'tick %.4f' % d['ms_per_step'], 'e2e %.4f' % d['e2e']['ms_per_step'], ' '.join('%s %.4f' % (k, v) for k, v in p.items() if k.startswith('edt')))"
  done
done
(cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 >/dev/null 2>&1)
