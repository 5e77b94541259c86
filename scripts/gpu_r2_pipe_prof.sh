# per-phase-kernel times and occupancy of the pipeline launches of one config-4 step (half scale)
timeout 900 ncu -k regex:pipe_ --clock-control none -s ${1:-240} -c ${2:-72} --csv \
  --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_blocks \
  --log-file gpurun_out/pipe_launches.csv python scripts/probe_config4.py --scale 0.5 --steps 3 > gpurun_out/pipe_prof.log 2>&1
echo rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/pipe_launches.csv") if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[ii], {"k": r[ki].split("(")[0].replace("void ttdvm::g32::", "").replace("void g32::", "")})
    try: d[r[mi]] = float(r[vi].replace(",", ""))
    except Exception: pass
print("| id | kernel | grid | us | regs | smem KB | warps act % | issue act % | fp64 % | Minst | occ lim reg/smem/blk | DRAM KB/output |")
for i, d in L.items():
    print("| %s | %s | %d | %.1f | %d | %.1f | %.1f | %.1f | %.1f | %.1f | %d/%d/%d | %.2f |" % (
        i, d["k"], d.get("launch__grid_size", 0), d.get("gpu__time_duration.sum", 0) / 1e3,
        d.get("launch__registers_per_thread", 0), d.get("launch__shared_mem_per_block_dynamic", 0) / 1024,
        d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
        d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
        d.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 0),
        d.get("smsp__inst_executed.sum", 0) / 1e6, d.get("launch__occupancy_limit_registers", 0),
        d.get("launch__occupancy_limit_shared_mem", 0), d.get("launch__occupancy_limit_blocks", 0),
        (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1024 / max(1, d.get("launch__grid_size", 1))))
PY
