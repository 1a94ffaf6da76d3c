"""Print registers / spills per kernel from an nvcc -Xptxas -v build log."""
import re
import sys

for path in sys.argv[1:]:
    lines = open(path).read().splitlines()
    for i, l in enumerate(lines):
        if "Compiling entry function" in l:
            name = re.search(r"'(\S+)'", l).group(1)
            blk = " ".join(lines[i:i + 5])
            regs = re.search(r"Used (\d+) registers", blk)
            sp = re.search(r"(\d+) bytes spill stores", blk)
            print(f"{name[:70]:70s} regs={regs and regs.group(1)} spill={sp and sp.group(1)}")
