"""Single-warp in-order latency model of a SASS loop body: the cycles one
warp needs per loop trip when only its own dependencies (and FP64 issue every
2 cycles) limit it, and the critical chain.
    cuobjdump -sass -fun K obj | python tools/sass_sim.py [min_len max_len]"""
import re
import sys
from collections import defaultdict

LAT = {"DFMA": 8, "DMUL": 8, "DADD": 8, "DSETP": 8, "MUFU": 18, "SHFL": 28, "LDS": 29, "LDC": 12, "LDCU": 12,
       "F2F": 10, "I2F": 10, "F2I": 10, "LDG": 300, "S2R": 20, "S2UR": 20, "R2UR": 6, "ATOMG": 300, "POPC": 6,
       "FLO": 6, "SYNCS": 60}
FP64 = {"DFMA", "DMUL", "DADD", "DSETP"}
lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (800, 1300)
ins = []
for l in sys.stdin.read().splitlines():
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: k for k, (a, _) in enumerate(ins)}
best = None
for k, (a, t) in enumerate(ins):
    m = re.search(r'\bBRA\b.*?(0x[0-9a-f]+)', t)
    if m:
        tg = int(m.group(1), 16)
        if tg < a and tg in addr and lo < k - addr[tg] < hi:
            best = (addr[tg], k)
b0, b1 = best
body = [t for _, t in ins[b0:b1 + 1]]


def regs(tok, wide):
    out = []
    m = re.match(r'-?\|?(R\d+)', tok)
    if m:
        r = int(m.group(1)[1:])
        out.append(r)
        if wide:
            out.append(r + 1)
    return out


def parse(t):
    s = t
    pred = None
    if s.startswith('@'):
        pred, s = s.split(' ', 1)
    op, _, rest = s.partition(' ')
    base = op.split('.')[0]
    wide = base in FP64 or '.64' in op or base in ("MUFU",) and '64' in op
    args = [a.strip() for a in rest.split(',')] if rest else []
    dst, src = [], []
    if base in ("STG", "STS", "ST", "BRA", "BSSY", "BSYNC", "SYNCS", "UTMALDG", "EXIT", "NOP", "YIELD", "BAR",
                "WARPSYNC", "ELECT", "UMOV", "UIADD3", "ULEA", "VOTEU"):
        for a in args:
            src += regs(a.replace('[', '').split('+')[0], True)
        return base, [], src
    if args:
        d = args[0]
        dwide = wide and base not in ("DSETP",)
        dst = regs(d, dwide and base != "F2F" or (base == "F2F" and "F64.F32" in op))
        for a in args[1:]:
            a2 = a.replace('[', '').replace(']', '')
            for piece in re.split(r'[+ ]', a2):
                src += regs(piece, wide)
    return base, dst, src


avail = defaultdict(int)
t_issue = 0
last_fp64 = -10
chain = {}
for trip in range(2):
    start = t_issue
    for idx, t in enumerate(body):
        base, dst, src = parse(t)
        ready = max([avail[r] for r in src] + [0])
        issue = max(ready, t_issue + 1)
        if base in FP64:
            issue = max(issue, last_fp64 + 2)
            last_fp64 = issue
        t_issue = issue
        lat = LAT.get(base, 5)
        for r in dst:
            avail[r] = issue + lat
    if trip == 1:
        dur = t_issue - start
n_fp64 = sum(1 for t in body if parse(t)[0] in FP64)
print(f"loop body: {len(body)} instructions, {n_fp64} fp64; one warp alone: {dur} cycles per trip "
      f"(issue-bound floor {max(len(body), 2 * n_fp64)})")
