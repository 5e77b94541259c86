# phase pipeline: parity suite with the pipeline forced on every eligible bin, then default; same-box A/B
TTDVM_PIPE_MIN=1 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash scripts/gpu_ab_env.sh TTDVM_PIPE=0 TTDVM_PIPE=1 TTDVM_PIPE=0 TTDVM_PIPE=1
