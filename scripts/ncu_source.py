"""Top SASS lines by stall samples for kernel #idx of an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]; want = int(sys.argv[2]) if len(sys.argv) > 2 else 0; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address":
        cur["h"] = r; continue
    if cur is not None and r:
        cur["rows"].append(r)
b = blocks[want]
h = b["h"]; idx = {n: i for i, n in enumerate(h)}
S = idx["Warp Stall Sampling (All Samples)"]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in b["rows"] if len(r) == len(h) and r[S].isdigit()]
tot = sum(int(r[S]) for r in data)
print(b["name"][:100], "samples", tot)
print("ALL", {c[6:]: sum(int(r[idx[c]] or 0) for r in data) for c in cols if sum(int(r[idx[c]] or 0) for r in data) > 0})
order = sorted(range(len(data)), key=lambda k: -int(data[k][S]))[:top]
for k in sorted(order):
    r = data[k]
    print(str(k).rjust(4), r[S].rjust(6), r[idx["Source"]][:70].ljust(70), {c[6:]: r[idx[c]] for c in cols if r[idx[c]] not in ("0", "")})
