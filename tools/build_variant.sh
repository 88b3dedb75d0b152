#!/bin/bash
# build an experimental liblbmgpu variant: tools/build_variant.sh NAME [nvcc -D flags...]
# (the device header can be swapped with LBM_DEVICE_HDR=/path/to/lbm_device.cuh, the AoS
# window source with LBM_AOS_SRC=/path/to/kernels_aos.cu)
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1111_0922_b200/csrc
OUT=$ROOT/build/variants/$NAME
rm -rf $OUT; mkdir -p $OUT/src
cp $SRC/*.cu $SRC/*.h $SRC/*.cuh $OUT/src/
if [ -n "$LBM_DEVICE_HDR" ]; then cp "$LBM_DEVICE_HDR" $OUT/src/lbm_device.cuh; fi
if [ -n "$LBM_AOS_SRC" ]; then cp "$LBM_AOS_SRC" $OUT/src/kernels_aos.cu; fi
mkdir -p $OUT/include; cp $ROOT/include/lbmgpu.h $OUT/include/
sed -i "s|../../include/lbmgpu.h|../include/lbmgpu.h|" $OUT/src/runtime.h
for f in kernels_direct kernels_aos kernels_indirect kernels_util kernels_swap kernels_swap1 kernels_aos_fb steppers slabs capi; do
  /usr/local/cuda/bin/nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
    -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin /usr/bin/g++ "$@" -c $OUT/src/$f.cu -o $OUT/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/liblbmgpu.so $OUT/*.o
echo $OUT/liblbmgpu.so
