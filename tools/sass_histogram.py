"""Static SASS opcode histogram of the headline kernel (the cfg2 default walk)
from the built object: python tools/sass_histogram.py > profiles/rNN_headline_sass_histogram.csv"""
import collections, pathlib, re, subprocess
ROOT = pathlib.Path(__file__).resolve().parent.parent
obj = ROOT / "paper_2205_01598_b200" / "csrc" / "build" / "mpk_lean_re.o"
fun = "_ZN4lmpk15mpk_lean_kernelILb0ELb1ELb1ELb0ELi4ELb0ELb0EEEvNS_9MpkParamsENS_11PowerCfgDevENS_10LeanParamsE"
out = subprocess.run(["cuobjdump", "-sass", "-fun", fun, str(obj)], capture_output=True, text=True).stdout
ops = collections.Counter()
for line in out.splitlines():
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if m:
        ops[m.group(1)] += 1
print("# SASS opcode histogram of the headline kernel (static instruction counts; cuobjdump -sass of")
print("# mpk_lean_kernel<CPLX=0, EXACT=1, VD=1, GEN=0, NP=4, XP=0, DP=0>, the cfg2 default walk, sm_100a).")
print("# TMA bulk copies: UBLKCP; mbarrier: SYNCS.*; FP64: DMUL/DADD (EXACT row sums); no tensor-core ops")
print("# (bandwidth-bound irregular gather). Dynamic counts per call are in r02_cfg2_ncu.txt / DESIGN.md 3.")
print(f"# {sum(ops.values())} instructions")
print("opcode,count")
for k, v in ops.most_common():
    print(f"{k},{v}")
