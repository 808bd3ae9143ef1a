#!/bin/bash
# Rebuild libvx.so with extra -D flags per variant and time dense EDTs
# (tools/edt_time.py); the default build is restored last.
#   tools/variant_edt.sh "base:" "rev:-DVX_P2_REVERSE_DENSE=1"
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  (cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 EXTRA="$flags" >/dev/null 2>&1) || { echo "$name: build failed"; continue; }
  python tools/edt_time.py 512 0.02 0 256 0.02 0 1024 0.02 0 512 0.0001 1 | sed "s/^/$name /"
done
(cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 >/dev/null 2>&1)
