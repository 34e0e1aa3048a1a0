"""Per-source-line instruction counts and stall samples of one kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next((r for r in rows if r and r[0] == "Line No"), None)
ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
f, res = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No", ""):
        continue
    try:
        res.append((int(r[ie]), float(r[ws]), f, r[0], r[1].strip()[:90]))
    except (ValueError, IndexError):
        pass
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"total warp instructions {ti}")
for n, s, f, ln, t in sorted(res, reverse=True)[:top]:
    print(f"{100 * n / ti:5.1f}% instr {100 * s / ts:5.1f}% stall  {f}:{ln}  {t}")
