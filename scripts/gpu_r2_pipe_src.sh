# source-line instruction counts of the LONGEST launch of one kernel (arg1: kernel regex; arg2/3: launch skip/count; arg4: steps) in config-4 steps (half scale)
REP=/tmp/pipe_src.ncu-rep
rm -f $REP
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${1:-pipe_gram1} -s ${2:-12} -c ${3:-12} -o ${REP%.ncu-rep} \
  python scripts/probe_config4.py --scale 0.5 --steps ${4:-3} > gpurun_out/pipe_src_cap.log 2>&1
echo rc=$?
ncu -i $REP --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size > /tmp/l.csv 2>&1
B=$(python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/l.csv")))
hdr = rows[0]; ti = hdr.index("gpu__time_duration.sum")
data = [r for r in rows[2:] if len(r) > ti]
best = max(range(len(data)), key=lambda i: float(data[i][ti].replace(",", "")))
import sys
sys.stderr.write("longest launch %d: %s\n" % (best, data[best][-2:]))
print(best)
PY
)
ncu -i $REP --page source --csv --print-source=cuda,sass --launch-skip $B --launch-count 1 > /tmp/src.csv 2>&1
python - <<'PY'
import csv
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
        res.append((g("Instructions Executed"), g("Warp Stall Sampling (All Samples)"), fname, int(r[0]), r[1][:100]))
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"instructions executed {ti:.0f}, samples {ts:.0f}")
for i, s, f, ln, src in sorted(res, reverse=True)[:40]:
    print(f"{100*i/ti:5.1f}% inst {100*s/ts:5.1f}% samp {f}:{ln} {src}")
PY
