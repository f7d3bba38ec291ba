#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of the built library (cuobjdump -sass;
runs without a GPU).  Proves which hardware paths each kernel uses:
DMMA (FP64 tensor), UTCxMMA (tcgen05), UBLKCP / UBLKPF (bulk-copy engine),
UTMALDG (tensor-map TMA), LDGSTS (cp.async), SYNCS (mbarriers), ...

    python scripts/sass_histogram.py [lib.so] > profiles/r02/sass_histogram.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("DMMA", "DFMA", "DMUL", "DADD", "HMMA", "UTCMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM",
        "UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "UTMAPF", "LDGSTS", "LDGDEPBAR", "SYNCS", "BAR", "LDS", "STS",
        "LDG", "STG", "ATOMG", "RED", "SHFL", "MUFU")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2303_04390_b200", "lib", "libphylograd.so")
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out = {}
    fn, hist = None, None
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            hist = out.setdefault(fn, collections.Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m and hist is not None:
            op = m.group(1)
            hist["_total"] += 1
            for k in KEYS:
                if op == k or (k in ("UTCMMA", "UTCHMMA", "UTCQMMA") and op.startswith("UTC") and "MMA" in op and op == k):
                    hist[k] += 1
            if op.startswith("UTC") and "MMA" in op:
                hist["UTC*MMA"] += 1
    demangled = {}
    names = list(out)
    try:
        dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    except Exception:
        dm = names
    for n, d in zip(names, dm):
        demangled[d] = {k: v for k, v in sorted(out[n].items()) if v}
    json.dump({"library": os.path.relpath(lib, ROOT), "tool": "cuobjdump -sass (CUDA 12.9)",
               "kernels": demangled}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
