"""Top CUDA source lines by warp-stall samples from an ncu report.
    python tools/src_hot.py <report> [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; res = []
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if len(r) > 8 and r[2] == "-":  # CUDA line rows carry '-' in the SASS address column
        try: s = int(r[4] or 0); n = int(r[7] or 0)
        except ValueError: continue
        res.append((s, n, f"{cur}:{r[0]}", r[1][:100]))
tot = sum(x[0] for x in res) or 1
for s, n, loc, src in sorted(res, reverse=True)[:N]:
    print(f"{100 * s / tot:5.1f}%  inst {n:>11d}  {loc:22s} {src}")
