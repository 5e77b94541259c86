# Build libttdvm_cuda.so of git revision $1 into build_ab/libttdvm_cuda_$2.so
# (A/B timing against the working tree: TTDVM_LIB=build_ab/... python ...).
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_1912_04582_b200/csrc include | tar -x -C "$TMP"
mkdir -p "$ROOT/build_ab"  # NB: listed in .gpurunignore; copy the .so under paper_1912_04582_b200/ab/ to ship it
OBJS=""
for f in "$TMP"/paper_1912_04582_b200/csrc/*.cu; do
  o="${f%.cu}.o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -c "$f" -o "$o" &
  OBJS="$OBJS $o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o "$ROOT/build_ab/libttdvm_cuda_$NAME.so"
rm -rf "$TMP"
echo "$ROOT/build_ab/libttdvm_cuda_$NAME.so"
