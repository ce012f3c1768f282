"""Aggregate an ncu source page (cuda,sass CSV) into the hottest CUDA lines with their top stall reasons."""
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
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            s = int(r[4])
        except ValueError:
            continue
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and not h.endswith("_not_issued"):
                try:
                    v = int(r[i])
                except ValueError:
                    continue
                if v:
                    stalls.append((v, h[6:]))
        stalls.sort(reverse=True)
        out.append((s, fname, r[0], r[1][:70], " ".join(f"{n}:{v}" for v, n in stalls[:3])))
tot = sum(o[0] for o in out) or 1
for s, f, l, src, st in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{l:<5} {src:<70} {st}")
