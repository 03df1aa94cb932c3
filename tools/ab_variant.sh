#!/bin/bash
# Developer A/B builds of one kernel file: compiles SRC (default csrc/sigma_ab.cu) with extra nvcc
# flags and links it with the other objects of the last full build into ablibs/libsbg_<name>.so.
#   tools/ab_variant.sh <name> "<nvcc flags>" [src.cu] [object-to-replace]
#   SBG_LIB_PATH=ablibs/libsbg_<name>.so python tools/sigma_modes.py c4
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; src=${3:-paper_2603_06101_b200/csrc/sigma_ab.cu}; base=${4:-sigma_ab}
mkdir -p ablibs build/ab
extra=""; [ "$base" = tables ] && extra="--fmad=false"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2603_06101_b200/csrc $extra $flags -c $src -o build/ab/${base}_$name.o
objs=$(ls build/sbg/*.o | grep -v "/${base}.o")
nccl=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'lib'))")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablibs/libsbg_$name.so $objs build/ab/${base}_$name.o \
  -L$nccl -l:libnccl.so.2 -Xlinker -rpath,$nccl
echo built ablibs/libsbg_$name.so
