"""Print registers / spills per kernel from the last build's ptxas log."""
import os
import re
import sys

log = open(os.path.join(os.path.dirname(__file__), "..", "paper_2310_17790_b200", "_build", "ptxas.log")).read()
cur = sp = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        sp = m.group(1)
    m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line) or re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{m.group(1):>4} regs spill {sp:>3}  {cur[:90]}")
        cur = None
