"""Registers / spills per kernel from `nvcc -Xptxas=-v` output on stdin (filter: argv[1] regex)."""
import re
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
fn = None
props = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and fn:
        props = f"stack {m.group(1)} spill st {m.group(2)} ld {m.group(3)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and fn:
        if pat is None or pat.search(fn):
            print(f"{m.group(1):>4} regs  {props:32s} {fn}")
        fn, props = None, ""
