# Same-box A/B of the face-factor kernel: base vs tiled-Gram build, timing and
# bitwise comparison of the outputs; GPU face-factor tests on the new build.
mkdir -p gpurun_out
A=paper_1912_04582_b200/ab/libttdvm_cuda_base.so; B=paper_1912_04582_b200/ab/libttdvm_cuda_ff1.so
for r in 1 2; do
  TTDVM_LIB=$A timeout 900 python scripts/ab_ff.py 8192 /tmp/ffA.npz >> gpurun_out/ab_ff.log 2>&1
  TTDVM_LIB=$B timeout 900 python scripts/ab_ff.py 8192 /tmp/ffB.npz >> gpurun_out/ab_ff.log 2>&1
done
python - >> gpurun_out/ab_ff.log 2>&1 <<'PY'
import numpy as np
a = np.load("/tmp/ffA.npz"); b = np.load("/tmp/ffB.npz")
for k in a.files:
    print(k, "bitwise equal" if a[k].shape == b[k].shape and np.array_equal(a[k], b[k], equal_nan=True) else "DIFFERENT")
PY
TTDVM_LIB=$B timeout 900 python -m pytest tests -x -q -m gpu -k "face or obstacle or wall" > gpurun_out/ab_ff_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_ff_tests.log
TTDVM_LIB=$B timeout 900 ncu --set full --clock-control none --import-source on -k regex:face_factor -s 1 -c 1 -o gpurun_out/prof_ff1 python scripts/probe_ff.py 1184 > gpurun_out/ncu_ff1.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_ff1.log
