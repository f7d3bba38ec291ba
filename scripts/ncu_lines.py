"""Per-source-line summary of an ncu report (instructions executed, stall samples).

usage: python scripts/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "traverse"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, hdr = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        ie = int(r[hdr["Instructions Executed"]] or 0)
        ss = int(r[2 + 2] or 0)
    except (ValueError, IndexError):
        continue
    res.append((ss, ie, fname, r[0], r[1].strip()[:90]))
tot_s = sum(x[0] for x in res) or 1
tot_i = sum(x[1] for x in res) or 1
print(f"total stall samples {tot_s}, instructions {tot_i}")
for ss, ie, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100*ss/tot_s:5.1f}% {100*ie/tot_i:5.1f}%i {f}:{ln:5s} {src}")
