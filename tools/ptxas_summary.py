"""Summarise `nvcc -Xptxas -v` output: registers / spills / stack per kernel."""
import re, subprocess, sys
out = subprocess.run([sys.executable, "-m", "paper_1203_5004_b200.build", "--verbose", "--force"],
                     capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1).replace("_ZN9hood_b200", "")
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack, st, ld = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if len(sys.argv) < 2 or re.search(sys.argv[1], cur):
            print(f"{cur[:70]:70s} regs={m.group(1):>4} stack={stack:>4} spill={st}/{ld}")
        cur = None
