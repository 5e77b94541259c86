# On the GPU box: full-set ncu capture of the rounding launches of one
# config-4 step (scale $1), then per-launch summary + source-line stalls of
# the longest launch, written as text under gpurun_out/ (the report itself
# stays on the box: it exceeds gpurun's copy-back limit).
set -u
SCALE=${1:-0.5}
SKIP=${2:-30}
CNT=${3:-12}
mkdir -p gpurun_out
REP=/tmp/prof_round.ncu-rep
rm -f $REP
timeout 1300 ncu --set full --clock-control none --import-source on -k regex:round_gram -s $SKIP -c $CNT \
  -o ${REP%.ncu-rep} python scripts/probe_config4.py --scale $SCALE --steps 4 > gpurun_out/ncu_cap.log 2>&1
echo "capture rc=$?"
ncu -i $REP --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/ncu_launches.csv 2>&1
python scripts/summarize_ncu.py --report $REP --out gpurun_out/ncu_sum > gpurun_out/ncu_summary.log 2>&1
python - <<'PY' > gpurun_out/ncu_longest.txt 2>&1
import csv, subprocess
rows = list(csv.reader(open("gpurun_out/ncu_launches.csv")))
hdr = rows[0]
ti = hdr.index("gpu__time_duration.sum")
data = [r for r in rows[2:] if len(r) > ti]
best = max(range(len(data)), key=lambda i: float(data[i][ti].replace(",", "")))
print("longest launch index", best, dict(zip(hdr, data[best])))
open("/tmp/best_id", "w").write(str(best))
PY
B=$(cat /tmp/best_id)
python scripts/ncu_stalls.py $REP "round_gram" 40 > gpurun_out/ncu_stalls_all.txt 2>&1
ncu -i $REP --page source --csv --print-source=cuda,sass --launch-skip $B --launch-count 1 -k regex:round_gram > /tmp/src_best.csv 2>&1
python - <<'PY' > gpurun_out/ncu_src_best.txt 2>&1
import csv, io
rows = list(csv.reader(open("/tmp/src_best.csv")))
fname, hdr, res = "", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        def g(name):
            try:
                return float(r[hdr.index(name)])
            except Exception:
                return 0.0
        res.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), fname, int(r[0]), r[1][:90]))
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
print("columns:", hdr)
print(f"total samples {ts:.0f}, instructions executed {ti:.0f}")
print("== by stall samples")
for s, i, f, ln, src in sorted(res, reverse=True)[:60]:
    print(f"{100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst {f}:{ln} {src}")
print("== by instructions executed")
for s, i, f, ln, src in sorted(res, key=lambda x: -x[1])[:40]:
    print(f"{100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst {f}:{ln} {src}")
PY
ls -la gpurun_out
