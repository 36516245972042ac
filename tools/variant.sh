#!/bin/bash
# Build a variant of libtrim_b200.so that differs only in the kernel
# instantiation TU(s) (trim_inst_<M>.o) by extra -D flags:
#   ./tools_variant.sh NAME "XFLAGS" [Ms...]   -> paper_2508_17828_b200/libtrim_b200_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; XF=$2; shift 2; MS=${@:-48}
C=paper_2508_17828_b200/csrc; O=build/obj; V=build/obj_$NAME
mkdir -p $V
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr"
OBJS="$O/trim_capi.o $O/trim_multi.o $O/trim_build.o $O/trim_graph.o"
for m in 16 32 48 120 0; do
  if [[ " $MS " == *" $m "* ]]; then
    nvcc $FLAGS $XF -DTRIM_M=$m -c -o $V/trim_inst_$m.o $C/trim_inst.cu 2> $V/trim_inst_$m.o.ptxas &
    OBJS="$OBJS $V/trim_inst_$m.o"
  else
    OBJS="$OBJS $O/trim_inst_$m.o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2508_17828_b200/libtrim_b200_$NAME.so $OBJS -ldl
echo built paper_2508_17828_b200/libtrim_b200_$NAME.so
