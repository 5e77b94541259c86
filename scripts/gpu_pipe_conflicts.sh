# shared-memory bank conflicts per source line of the six pipeline kernels (one chunk) in a config-4 step (half scale)
#   gpurun -- 'bash scripts/gpu_pipe_conflicts.sh [skip] [count] [steps] [regex]'
REP=/tmp/pipe_conf.ncu-rep
if [ -z "$REUSE" ]; then
rm -f $REP
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${4:-pipe_} -s ${1:-60} -c ${2:-6} -o ${REP%.ncu-rep} \
  python scripts/probe_config4.py --scale 0.5 --steps ${3:-3} > gpurun_out/pipe_conf_cap.log 2>&1
echo rc=$?
fi
for L in $(seq 0 $((${2:-6} - 1))); do
ncu -i $REP --page source --csv --print-source=cuda,sass --launch-skip $L --launch-count 1 > /tmp/src.csv 2>&1
ncu -i $REP --page raw --csv --launch-skip $L --launch-count 1 --metrics gpu__time_duration.sum,launch__grid_size,smsp__inst_executed.sum > /tmp/raw.csv 2>&1
python - <<'PY'
import csv
raw = list(csv.reader(open("/tmp/raw.csv")))
try:
    h = raw[0]; r = raw[2]
    print("== launch", r[h.index("Kernel Name")][:60], "grid", r[h.index("launch__grid_size")], "us", r[h.index("gpu__time_duration.sum")])
except Exception as e:
    print("== launch ?", e)
rows = list(csv.reader(open("/tmp/src.csv")))
fname, hdr, res = "", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        def g(name):
            try: return float(r[hdr.index(name)])
            except Exception: return 0.0
        res.append((g("L1 Wavefronts Shared Excessive"), g("L1 Wavefronts Shared"), g("Instructions Executed"),
                    g("Warp Stall Sampling (All Samples)"), fname, int(r[0]), r[1][:90]))
tx = sum(x[0] for x in res); tw = sum(x[1] for x in res) or 1; ti = sum(x[2] for x in res) or 1; ts = sum(x[3] for x in res) or 1
print(f"shared wavefronts {tw:.3g}, excessive {tx:.3g} ({100*tx/tw:.1f} %), instructions {ti:.3g}")
for x, w, i, s, f, ln, src in sorted(res, reverse=True)[:8]:
    if x <= 0: break
    print(f"  excess {100*x/tw:5.1f}% of wavefronts (line total {100*w/tw:5.1f}%) inst {100*i/ti:4.1f}% samp {100*s/ts:4.1f}%  {f}:{ln} {src}")
print("  -- top by stall samples")
for x, w, i, s, f, ln, src in sorted(res, key=lambda t: -t[3])[:8]:
    print(f"  samp {100*s/ts:4.1f}% inst {100*i/ti:4.1f}%  {f}:{ln} {src}")
PY
done
