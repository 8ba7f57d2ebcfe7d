#!/bin/bash
# Build an experiment variant of libpba_gpu.so: tools/build_variant.sh NAME "-DFOO=1 ..."
# Output: paper_1704_06967_b200/lib/variants/NAME.so (selected with PBA_GPU_LIB; experiments only).
set -e
cd "$(dirname "$0")/../paper_1704_06967_b200/csrc"
name=$1; shift
make -s -j8 OUT=../lib/variants/_$name NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $*"
cp ../lib/variants/_$name/libpba_gpu.so ../lib/variants/$name.so
rm -rf ../lib/variants/_$name
echo "built lib/variants/$name.so"
