# round-2 evidence: compute-sanitizer runs, ncu launch list of the bench command, full-set capture of the rounding launches
set -u
mkdir -p gpurun_out/r02
python scripts/sanitize_small.py > gpurun_out/r02/sanitize_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 python scripts/sanitize_small.py > gpurun_out/r02/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02/sanitize_$tool.log
done
# launch list of the bench command (per-launch times are cold-cache and serialised: shares only)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02/launches_bench.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/r02/ncu_bench.log 2>&1
echo "launch list rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/r02/launches_bench.csv") if l.startswith('"')))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    try: v = float(r[vi].replace(",", ""))
    except Exception: continue
    name = r[ki].split("(")[0]
    tot[name] += v; cnt[name] += 1
s = sum(tot.values())
with open("gpurun_out/r02/launches_bench.md", "w") as f:
    f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
    for k, v in tot.most_common():
        f.write(f"| `{k}` | {cnt[k]} | {v/1e6:.2f} | {100*v/s:.1f} % |\n")
print(open("gpurun_out/r02/launches_bench.md").read())
PY
bash scripts/ncu_box_round.sh 0.5 100 45 > gpurun_out/r02/ncu_round.log 2>&1; echo "round capture rc=$?"
cp gpurun_out/ncu_sum* gpurun_out/ncu_longest.txt gpurun_out/ncu_stalls_all.txt gpurun_out/ncu_src_best.txt gpurun_out/ncu_launches.csv gpurun_out/r02/ 2>/dev/null
ls gpurun_out/r02
