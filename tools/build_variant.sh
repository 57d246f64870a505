#!/bin/bash
# Build a variant of libsc_b200.so with extra nvcc defines for sc_graph.cu only (A/B probes):
#   tools/build_variant.sh NAME -DSC_MINB_W=6 ...   -> tools/variants/NAME/libsc_b200.so
# (load it with SC_LIB_PATH=tools/variants/NAME/libsc_b200.so)
set -e
cd "$(dirname "$0")/../paper_2310_10939_b200/csrc"
NAME=$1; shift
OUT=../../tools/variants/$NAME
mkdir -p $OUT
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-O3,-ffp-contract=off -Xptxas -v \
    --expt-relaxed-constexpr "$@" -c sc_graph.cu -o $OUT/sc_graph.o 2> $OUT/ptxas.log
OBJS=$(ls build/*.o | grep -v sc_graph.o)
$NV $ARCH -shared -o $OUT/libsc_b200.so $OUT/sc_graph.o $OBJS -lcudart_static -lrt -ldl -lpthread
grep -A2 "k_rw_step" $OUT/ptxas.log | grep -E "Compiling|registers" | paste - - | sed -E 's/.*k_rw_stepILb(.)ELb(.)ELb(.).*Used ([0-9]+) registers.*spill.*/U\1 S\2 F\3: \4 regs/' | head -3
grep -A3 "k_rw_step" $OUT/ptxas.log | grep -i spill | head -3
