# A/B of environment switches on the config-3 microbench (resident inputs).
mkdir -p gpurun_out
for env in "$@"; do
  echo "== $env"
  env $env timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
