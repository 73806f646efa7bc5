#!/bin/bash
# build an experimental libvdmc variant (profiling build: -DVDMC_PROFILING):
#   tools/build_variant.sh NAME 'sed-expression-on-enum.cu'
set -e
NAME=$1; EXPR=$2
D=/tmp/vdmc_variant_$NAME; rm -rf $D; mkdir -p $D/csrc
cp paper_2201_11655_b200/csrc/*.cu paper_2201_11655_b200/csrc/*.cuh $D/csrc/
sed -i "$EXPR" $D/csrc/enum.cu
sed -i 's#"../../include/vdmc.h"#"/root/repo/include/vdmc.h"#' $D/csrc/vdmc_internal.cuh
NCCL=$(python -c "import paper_2201_11655_b200.build as b; print(b.NCCL)")
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DVDMC_PROFILING -I$NCCL/include"
for f in api build enum enum32 edges layers; do nvcc $F -c -o $D/$f.o $D/csrc/$f.cu & done
for j in $(jobs -p); do wait $j || { echo "compile failed"; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2201_11655_b200/lib/libvdmc_$NAME.so $D/*.o \
    -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo built paper_2201_11655_b200/lib/libvdmc_$NAME.so
