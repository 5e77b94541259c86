TTDVM_PIPE_MIN=1 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python -m pytest tests -m gpu -q 2>&1 | tail -3
bash scripts/gpu_ab_env.sh TTDVM_PIPE_KEEPMS=0 TTDVM_PIPE_KEEPMS=1 TTDVM_PIPE_KEEPMS=0 TTDVM_PIPE_KEEPMS=1
