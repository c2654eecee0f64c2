"""Per-source-line instruction counts of an ncu capture (run here): python scripts/src_lines.py rep [per] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
per = float(sys.argv[2]) if len(sys.argv) > 2 else 378450
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
for i, r in enumerate(rows):
    if r and r[0] == "Line No":
        hdr, start = r, i + 1
        break
ie = hdr.index("Instructions Executed")
tot, lines = 0, []
for r in rows[start:]:
    if len(r) > ie and r[0].isdigit() and r[2] == '-':
        try:
            v = int(r[ie])
        except ValueError:
            continue
        lines.append((v, int(r[0]), r[1][:100]))
        tot += v
print(f"total {tot} = {tot / per:.1f} per unit")
for v, l, src in sorted(lines, reverse=True)[:top]:
    print(f"{v / per:8.1f} {l:5d} {src}")
