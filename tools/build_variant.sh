#!/bin/bash
# build an experimental variant of libovs.so: tools/build_variant.sh <name> "<nvcc -D flags>"
# -> tools/vso/libovs_<name>.so (every translation unit; the flags select code paths under test)
set -e
NAME=$1; FLAGS=$2
D=/root/repo/tools/variants/$NAME; mkdir -p $D
C=${SRC:-/root/repo/paper_1608_08648_b200/csrc}
NC=$(python -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
ARCH="-gencode arch=compute_100a,code=sm_100a"
# ONLY="ovs_u32_k ..." compiles just those units with the flags and links the in-tree build's other objects
ALL="ovs_api ovs_host ovs_dist ovs_s32_k ovs_u32_k ovs_u32_v ovs_i32_k ovs_i32_v ovs_f64_k ovs_f64_v"
for f in $ALL; do
  if [ -n "$ONLY" ] && ! echo " $ONLY " | grep -q " $f "; then cp $C/build/$f.o $D/$f.o; continue; fi
  nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -I/root/repo/include -I$NC/include $FLAGS -c -o $D/$f.o $C/$f.cu &
done
wait
mkdir -p /root/repo/tools/vso; nvcc $ARCH -shared -o /root/repo/tools/vso/libovs_$NAME.so $D/*.o -L$NC/lib -l:libnccl.so.2 -Xlinker -rpath=$NC/lib
rm -rf $D
echo built libovs_$NAME.so
