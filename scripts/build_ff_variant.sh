# Rebuild only facefactor.cu with extra nvcc flags and link it with the in-tree objects into
# paper_1912_04582_b200/ab/libttdvm_cuda_$1.so (A/B via TTDVM_LIB).
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1912_04582_b200/csrc
mkdir -p "$ROOT/paper_1912_04582_b200/ab"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr "$@" -c $C/facefactor.cu -o /tmp/facefactor_$NAME.o
OBJS=$(ls $C/*.o | grep -v facefactor.o)
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS /tmp/facefactor_$NAME.o \
  -o "$ROOT/paper_1912_04582_b200/ab/libttdvm_cuda_$NAME.so"
cuobjdump -res-usage /tmp/facefactor_$NAME.o 2>&1 | grep -A1 "face_factor_kernelILi1" | tail -1 | cut -c1-60
