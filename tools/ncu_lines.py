"""Per-source-line stall breakdown from an ncu report (cuda,sass source view).

    python tools/ncu_lines.py report.ncu-rep [top_n] [line_lo line_hi]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
for i, r in enumerate(rows[:10]):
    if "Warp Stall Sampling (All Samples)" in r:
        hdr, st = r, i + 1
        break
reasons = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in reasons}
iall = hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: collections.Counter())
text = {}
tot = 0
for r in rows[st:]:
    if len(r) <= iall or not r[0]:
        continue
    try:
        ln = int(r[0])
        s = int(r[iall])
    except ValueError:
        continue
    if not lo <= ln <= hi:
        continue
    text[ln] = r[1].strip()[:70]
    agg[ln]["all"] += s
    tot += s
    for c in reasons:
        try:
            agg[ln][c[6:]] += int(r[idx[c]])
        except ValueError:
            pass
print("total samples", tot)
for ln, c in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
    parts = ", ".join(f"{k}={v}" for k, v in c.most_common(5) if k != "all" and v)
    print(f"{c['all']:7d} {100 * c['all'] / max(tot, 1):5.1f}% L{ln}: {text[ln]}  [{parts}]")
