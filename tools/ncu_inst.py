"""Instructions executed per CUDA source line from an ncu source page (cuda,sass CSV)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
fname, hdr, out = "?", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            v = int(r[ie])
        except ValueError:
            continue
        out.append((v, fname, int(r[0]), r[1][:80]))
tot = sum(o[0] for o in out) or 1
print(f"total warp instructions {tot:.4g}")
for v, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l:<5} {src}")
