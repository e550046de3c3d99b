#!/bin/bash
# Same-box A/B helper: rebuild ONE translation unit with extra -D flags and
# link it with the other (already built) objects into ab_libs/<name>.so; load
# it with RP_LIB=ab_libs/<name>.so.  usage: build_variant.sh name unit.cu -DX=1 ...
set -e
NAME=$1; UNIT=$2; shift 2
PKG=paper_2604_27085_b200
mkdir -p ab_libs/obj_$NAME
OBJ=ab_libs/obj_$NAME/$(basename $UNIT).o
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
  -Xcompiler -fPIC,-fvisibility=hidden,-fvisibility-inlines-hidden -Iinclude -I$PKG/csrc \
  --expt-relaxed-constexpr -DROUNDPIPE_CONFIG_DIR=\"$(pwd)/configs\" -Xptxas -v "$@" \
  -c $PKG/csrc/kernels/$UNIT -o $OBJ 2> ab_libs/obj_$NAME/ptxas.log
# REPLACES: the built unit this variant stands in for (default: UNIT itself;
# e.g. REPLACES=elementwise.cu for a copy of an older elementwise.cu)
REPLACES=${REPLACES:-$UNIT}
OTHERS=$(find build -name '*.o' ! -name "$(basename $REPLACES).o")
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xlinker -Bsymbolic \
  -o ab_libs/$NAME.so $OBJ $OTHERS -lpthread -ldl
grep -A2 "qk_norm" ab_libs/obj_$NAME/ptxas.log | grep -E "Used|spill" | sed 's/ptxas info    ://' | paste - - | head
