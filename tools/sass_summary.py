"""Instruction-class counts per kernel of the built libadps.so (cuobjdump -sass), dev helper.

python tools/sass_summary.py "header" > profiles/rNN_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2605_06876_b200/libadps.so"
CLASSES = ["ACQBULK", "UBLKCP", "SYNCS", "LDGSTS", "REDUX", "MATCH", "VOTE", "SHFL", "ATOMS", "ATOMG", "RED",
           "BAR", "MUFU", "DFMA", "DADD", "DMUL", "HMMA", "UTCMMA", "UTCHMMA", "UCGABAR_ARV", "UCGABAR_WAIT", "ATOM"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts.setdefault(kern, collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if kern and m:
        op = m.group(1)
        for c in CLASSES:
            if op == c or op.startswith(c + "."):
                counts[kern][c] += 1
try:
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
except OSError:
    names = list(counts)
header = sys.argv[1] if len(sys.argv) > 1 else ""
if header:
    print(header)
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print(f"total over {len(counts)} kernels: {dict(tot)}")
for name, (k, c) in sorted(zip(names, counts.items())):
    print(f"{name[:100]:100s} {dict(c)}")
