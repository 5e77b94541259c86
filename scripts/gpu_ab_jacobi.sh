# Same-box A/B of the Jacobi stopping rule (TTDVM_JACOBI_BIG2) on the config-4
# half-scale probe, then the GPU suite on each looser build.
mkdir -p gpurun_out
D=paper_1912_04582_b200/ab
for r in 1 2; do
  for L in cur jb10 jb14; do
    echo "== $L" >> gpurun_out/ab_jac.log
    TTDVM_LIB=$D/libttdvm_cuda_$L.so timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 5 2>&1 | grep "\"step\": [2-5]" | cut -c1-600 >> gpurun_out/ab_jac.log
  done
done
for L in jb10 jb14; do
  TTDVM_LIB=$D/libttdvm_cuda_$L.so timeout 900 python -m pytest tests -q -m gpu > gpurun_out/ab_jac_tests_$L.log 2>&1; echo "rc=$?" >> gpurun_out/ab_jac_tests_$L.log
done
