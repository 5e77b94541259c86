"""SASS instructions per source line (code footprint) of a kernel in an ncu report."""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cnt, ex = collections.Counter(), collections.Counter()
fname, cur, hdr = "", None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        cur = (fname, int(r[0]), r[1][:70])
    elif hdr and r and r[0] == "" and len(r) > 3 and r[2].startswith("0x") and cur:
        cnt[cur] += 1
tot = sum(cnt.values())
print("SASS instructions attributed:", tot)
byf = collections.Counter()
for k, v in cnt.items():
    byf[k[0]] += v
print(byf.most_common())
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(v, f"{k[0]}:{k[1]}", k[2])
