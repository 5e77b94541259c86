# Build the working tree's library with extra nvcc flags into
# paper_1912_04582_b200/ab/libttdvm_cuda_$1.so (ships with gpurun; A/B via TTDVM_LIB).
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$(mktemp -d)
mkdir -p "$ROOT/paper_1912_04582_b200/ab"
OBJS=""
for f in "$ROOT"/paper_1912_04582_b200/csrc/*.cu; do
  o="$OUT/$(basename "${f%.cu}").o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr "$@" -c "$f" -o "$o" &
  OBJS="$OBJS $o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o "$ROOT/paper_1912_04582_b200/ab/libttdvm_cuda_$NAME.so"
cuobjdump -res-usage $OUT/round.o 2>&1 | grep -A1 "round_gram_kernelILi0ELb0" | tail -1 | cut -c1-60
rm -rf "$OUT"
