#!/bin/bash
# Cross-compile libvx.so variants with extra -D flags (tuning experiments):
#   tools/build_lib_variants.sh OUTDIR "name:-DFLAG=1 ..." ...
# -> OUTDIR/libvx_<name>.so; run one on the GPU box with VX_LIB=OUTDIR/libvx_<name>.so
cd "$(dirname "$0")/../paper_2407_02363_b200/csrc"
out=$1; shift
mkdir -p "$out"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr"
for v in "$@"; do
  (name=${v%%:*}; flags=${v#*:}; d=$(mktemp -d)
   $NV $flags -c vx_edt.cu -o $d/vx_edt.o 2>/dev/null &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libvx_$name.so" $d/vx_edt.o \
        $(ls _obj/*.o | grep -v vx_edt.o) -lcudart && echo "built $name") &
done
wait
