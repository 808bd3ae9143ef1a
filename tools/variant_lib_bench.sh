#!/bin/bash
# 512^3 camera tick and its phases per prebuilt library variant (GPU box):
#   tools/variant_lib_bench.sh DIR name1 name2 ...   (DIR/libvx_<name>.so, tools/build_lib_variants.sh)
cd "$(dirname "$0")/.."
dir=$1; shift
for rep in 1 2; do
  for name in "$@"; do
    VX_LIB=$dir/libvx_$name.so python bench.py --steps 400 --warmup 5 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); p=d['phase_ms']
print('%-8s' % '$name', 'tick %.4f' % d['ms_per_step'], 'e2e %.4f' % d['e2e']['ms_per_step'], ' '.join('%s %.4f' % (k, v) for k, v in p.items() if k.startswith('edt')))"
  done
done
