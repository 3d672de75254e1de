"""Instruction / stall histogram of an `ncu --page source --csv --print-source sass` export."""
import csv
import sys
from collections import Counter

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if r]
    hdr = next(r for r in rows if r[0] == "Address")
    data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr) and r[0] != "Address"]
    end = next((i for i, r in enumerate(data) if r[0] == "Kernel Name"), len(data))
    data = [r for r in data[:end] if r[hdr.index("Instructions Executed")].isdigit()]
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie] or 0) for r in data)
    st = sum(int(r[ss] or 0) for r in data)
    print(f, "warp instrs", tot, "samples", st)
    c, cs = Counter(), Counter()
    for r in data:
        t = r[1].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += int(r[ie] or 0)
        cs[op] += int(r[ss] or 0)
    print(" instrs ", c.most_common(16))
    print(" samples", cs.most_common(16))
    if "-v" in sys.argv[0:1] or len(sys.argv) > 2:
        for r in sorted(data, key=lambda r: -int(r[ss] or 0))[:20]:
            print("   ", r[0][-5:], r[ss], r[ie], r[1][:80])
