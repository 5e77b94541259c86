"""Per-line stall-reason breakdown (cuda,sass view) of an ncu report.
    python scripts/ncu_stalls.py report.ncu-rep kernel-regex [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname, agg, tot = None, "", {}, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    elif hdr and r and r[0].isdigit():
        key = (fname, int(r[0]), r[1][:70])
        d = agg.setdefault(key, {})
        for i in cols:
            try:
                v = int(r[i])
            except ValueError:
                continue
            d[hdr[i]] = d.get(hdr[i], 0) + v
            tot[hdr[i]] = tot.get(hdr[i], 0) + v
T = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for key, d in sorted(agg.items(), key=lambda x: -sum(x[1].values()))[:top]:
    s = sum(d.values())
    parts = ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3])
    print(f"{100*s/T:5.1f}% {key[0]}:{key[1]} {key[2]} [{parts}]")
