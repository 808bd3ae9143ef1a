#!/bin/bash
# Dense-EDT times and the 512^3 camera tick per prebuilt library variant (GPU box):
#   tools/variant_edt_bench.sh DIR name1 name2 ...   (DIR/libvx_<name>.so)
cd "$(dirname "$0")/.."
dir=$1; shift
for rep in 1 2; do
  for name in "$@"; do
    echo "== $name"
    VX_LIB=$dir/libvx_$name.so python tools/edt_time.py 512 0.02 0 1024 0.02 0 256 0.02 0
  done
done
