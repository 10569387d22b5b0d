"""Summarise -Xptxas -v logs: one line per kernel/function (regs, spills, stack)."""
import re, sys
for path in sys.argv[1:]:
    print("==", path)
    cur = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'|Function properties for (\S+)", line)
        if m:
            cur = m.group(1) or m.group(2)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            st, ss, sl = m.groups()
            print(f"  {cur[:90]:90s} stack {st:>4} spill {ss:>4}/{sl:>4}", end="")
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            print(f" regs {m.group(1)}")
            cur = None
