"""Summarise an ncu report's SASS page: instructions per cell by opcode.
    python tools/sass_mix.py <report.ncu-rep> <cells> [kernel-regex]"""
import collections, csv, io, subprocess, sys
rep, cells = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); iss = hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); st = collections.Counter(); tot = 0; tst = 0
for r in data:
    try: n = int(r[ia] or 0)
    except ValueError: continue
    toks = r[isrc].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    ops[op] += n; tot += n; s = int(r[iss] or 0); st[op] += s; tst += s
wc = cells / 32
print(f"warp-instructions per warp-cell (= thread instr per cell): {tot / wc:.1f}")
fp64 = sum(ops[o] for o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")) / wc
print(f"fp64 pipe per cell: {fp64:.1f}")
for op, n in ops.most_common(30):
    print(f"  {op:10s} {n / wc:7.1f}   stall% {100 * st[op] / max(tst, 1):5.1f}")
