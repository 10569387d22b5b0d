"""Per CUDA source line: executed SASS instructions per cell split by opcode.
    python tools/line_ops.py <report.ncu-rep> <cells> [N]"""
import collections, csv, io, subprocess, sys
rep, cells = sys.argv[1], float(sys.argv[2]); N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, cur_line = None, None
per = collections.defaultdict(collections.Counter)
src = {}
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0] != "":
        cur_line = f"{cur_file}:{r[0]}"; src[cur_line] = r[1][:80]; continue
    if len(r) < 9: continue
    try: n = int(r[7] or 0)
    except ValueError: continue
    sass = r[3].split()
    if not sass: continue
    op = sass[1] if sass[0].startswith('@') else sass[0]
    per[cur_line][op.split('.')[0] if not op.startswith('IMAD.MOV') else 'IMAD.MOV'] += n
wc = cells / 32
tot = sorted(((sum(c.values()), k) for k, c in per.items()), reverse=True)
allc = sum(t for t, _ in tot)
print(f"total thread-inst per cell {allc / wc:.1f}")
for t, k in tot[:N]:
    ops = ", ".join(f"{o} {v / wc:.1f}" for o, v in per[k].most_common(5))
    print(f"{t / wc:6.1f} {k:26s} {src.get(k, '')[:60]:60s} | {ops}")
