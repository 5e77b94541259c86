python -m pytest tests -m gpu -q -x 2>&1 | tail -4
TTDVM_XWIDE_D=24 TTDVM_PIPE_MIN=1 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash scripts/gpu_ab_env.sh TTDVM_XWIDE_D=0 TTDVM_XWIDE_D=40 TTDVM_XWIDE_D=32 TTDVM_XWIDE_D=24 TTDVM_XWIDE_D=0 TTDVM_XWIDE_D=40
for v in 0 32; do
  echo "== config 3 TTDVM_XWIDE_D=$v"
  TTDVM_XWIDE_D=$v python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(round(d['value']), 'tensors/s', round(d['roofline']['frac'], 4), 'of FP64 peak')"
done
for v in 0 40; do
  echo "== config 5 scale 0.25 TTDVM_XWIDE_D=$v"
  TTDVM_XWIDE_D=$v python bench.py --config 5 --scale 0.25 --steps 4 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(round(d['value']), 'cell-steps/s', {k: v['ms_per_step'] for k, v in d['roofline']['per_kernel'].items()})"
done
