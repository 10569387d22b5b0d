"""List the loops (backward branches) of one kernel's SASS with their instruction mix.
    cuobjdump -sass -fun <kernel> <obj> | python tools/sass_loops.py"""
import re, sys, collections
lines = sys.stdin.read().splitlines()
ins = []
for l in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: k for k, (a, _) in enumerate(ins)}
for k, (a, t) in enumerate(ins):
    m = re.search(r'\bBRA\b.*?(0x[0-9a-f]+)', t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr_idx:
        continue
    body = ins[addr_idx[tgt]:k + 1]
    ops = collections.Counter()
    for _, s in body:
        tok = s.split()
        op = tok[1] if tok[0].startswith('@') else tok[0]
        ops[op.split('.')[0]] += 1
    fp64 = sum(ops[o] for o in ('DFMA', 'DMUL', 'DADD', 'DSETP'))
    if len(body) < 100:
        continue
    print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, fp64 {fp64}, LDL {ops['LDL']}, STL {ops['STL']}, "
          f"SHFL {ops['SHFL']}, MUFU {ops['MUFU']}, MOV {ops['MOV'] + ops['IMAD']}, LDC {ops['LDC'] + ops['LDCU']}, BRA {ops['BRA']}")
