"""Per-kernel SASS instruction summary of libpi0b.so (cuobjdump -sass): the tcgen05 / TMA / TMEM
evidence for every kernel.  python scripts/sass_summary.py [lib] > profiles/r02_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2510_26742_b200", "libpi0b.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
# mnemonic families: tcgen05.mma (UTCHMMA / UTCQMMA...), tcgen05.ld/st (LDTM/STTM), TMA (UTMALDG /
# UTMASTG / UTMAPF), bulk copies (UBLKCP), mbarrier (SYNCS), legacy mma.sync (HMMA), cp.async (LDGSTS)
FAMS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "HMMA", "REDG", "RED", "ATOMG"]
kern = None
counts = collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts.setdefault(kern, collections.Counter())
        continue
    if kern is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op, suf = m.group(2), (m.group(3) or "")
        c = counts[kern]
        c["_total"] += 1
        for f in FAMS:
            if op == f or (f == "RED" and op.startswith("RED")):
                c[f] += 1
        if op == "UTCHMMA" and ".2CTA" in suf:
            c["UTCHMMA.2CTA"] += 1
print(f"SASS instruction families per kernel of {os.path.relpath(lib, ROOT)} (cuobjdump -sass)")
print("UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld (TMEM -> registers), UTMALDG = TMA tensor load, "
      "UBLKCP = bulk copy, SYNCS = mbarrier ops, LDGSTS = cp.async, HMMA = legacy mma.sync (must be 0)")
cols = ["_total", "UTCHMMA", "UTCHMMA.2CTA", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "HMMA", "RED"]
print(f"{'kernel':70s} " + " ".join(f"{c.strip('_'):>12s}" for c in cols))
tot = collections.Counter()
for k, c in counts.items():
    name = demangle(k)
    name = name if len(name) <= 70 else name[:67] + "..."
    print(f"{name:70s} " + " ".join(f"{c[x]:12d}" for x in cols))
    tot.update(c)
print(f"{'ALL':70s} " + " ".join(f"{tot[x]:12d}" for x in cols))
