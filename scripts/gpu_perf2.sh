python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash scripts/gpu_ab.sh X=cur
python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline | cut -c1-150
python bench.py --config 5 --scale 0.25 --steps 3 --warmup 3 --no-cpu-baseline | cut -c1-150
