# ncu launch list (gpu__time_duration only, no clock control) of the bench command; per-kernel shares of the step
# launches (set-up kernels listed separately).  Per-launch times are cold-cache and serialised: shares only.
mkdir -p gpurun_out/r02
timeout 2300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_bench_end.csv \
  python bench.py --steps ${1:-20} --warmup ${2:-3} --no-cpu-baseline --no-parity > gpurun_out/r02/ncu_bench_end.log 2>&1
echo "launch list rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/r02/launches_bench_end.csv") if l.startswith('"')))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    try: v = float(r[vi].replace(",", ""))
    except Exception: continue
    name = r[ki].split("(")[0]
    tot[name] += v; cnt[name] += 1
setup = {k for k in tot if any(s in k for s in ("face_factor", "xin_kernel", "dfma_probe"))}
s = sum(v for k, v in tot.items() if k not in setup)
with open("gpurun_out/r02/launches_bench_end.md", "w") as f:
    f.write("| kernel | launches | total ms | share of the step launches |\n|---|---|---|---|\n")
    for k, v in tot.most_common():
        share = "set-up" if k in setup else f"{100*v/s:.1f} %"
        f.write(f"| `{k}` | {cnt[k]} | {v/1e6:.2f} | {share} |\n")
print(open("gpurun_out/r02/launches_bench_end.md").read())
PY
# keep the raw list small: per-launch rows of the last 2000 launches only
(head -3 gpurun_out/r02/launches_bench_end.csv; grep '^"' gpurun_out/r02/launches_bench_end.csv | tail -2000) > gpurun_out/r02/launches_bench_end_tail2000.csv
rm -f gpurun_out/r02/launches_bench_end.csv
