"""Static control codes of a SASS loop body (sm_90/sm_100 128-bit encoding):
the sum of the stall counts ptxas put on each instruction is the cycles one
warp spends in fixed-latency waits per loop trip, before any variable-latency
(scoreboard) wait.
    cuobjdump -sass -fun K obj | python tools/sass_ctrl.py [min_len max_len]"""
import collections
import re
import sys

lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (400, 1300)
ins = []
lines = sys.stdin.read().splitlines()
for n, l in enumerate(lines):
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/', l)
    if m:
        m2 = re.search(r'/\* (0x[0-9a-f]+) \*/', lines[n + 1])
        ins.append((int(m.group(1), 16), m.group(2).strip(), int(m2.group(1), 16)))
addr = {a: k for k, (a, _, _) in enumerate(ins)}
loops = []
for k, (a, t, _) in enumerate(ins):
    m = re.search(r'\bBRA\b.*?(0x[0-9a-f]+)', t)
    if m:
        tg = int(m.group(1), 16)
        if tg < a and tg in addr and lo < k - addr[tg] < hi:
            loops.append((addr[tg], k))
b0, b1 = loops[-1]
tot = 0
by = collections.Counter()
cnt = collections.Counter()
for a, t, h in ins[b0:b1 + 1]:
    stall = (h >> 41) & 0xF
    s = t.split(' ', 1)[1] if t.startswith('@') else t
    op = s.split(' ')[0]
    tot += stall
    by[op] += stall
    cnt[op] += 1
n = b1 - b0 + 1
print(f"loop {b0}-{b1}: {n} instructions, static stall cycles {tot} ({tot / n:.2f} per instruction)")
for op, v in by.most_common(14):
    print(f"  {op:24s} n={cnt[op]:4d} stall={v:5d} avg={v / cnt[op]:.2f}")
