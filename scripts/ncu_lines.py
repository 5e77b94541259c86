"""Top source lines by warp-stall samples from an ncu report (cuda,sass view).
    python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = ""
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "File Path", "Function Name") and r[0].isdigit():
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        if s:
            res.append((s, fname, int(r[0]), r[1][:90]))
tot = sum(x[0] for x in res)
res.sort(reverse=True)
print(f"total samples {tot}")
for s, f, ln, src in res[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln} {src}")
