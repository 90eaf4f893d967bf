"""Print registers / spills per fused-kernel instance from the ptxas logs (build/)."""
import glob
import re

for path in sorted(glob.glob("build/ptxas_mcsf_inst_d*.cu.log")):
    cur = sp = None
    for line in open(path):
        m = re.search(r"CfgILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", line)
        if "Compiling entry" in line and m:
            cur = m.groups()
            continue
        if cur and "spill" in line:
            sp = re.sub(r"\s+", " ", line.strip())
        m2 = re.search(r"Used (\d+) registers", line)
        if m2 and cur:
            print("D=%s R=%s NA=%s KB=%s SH=%s" % cur, "regs", m2.group(1), sp)
            cur = None
