#!/usr/bin/env python
"""Parity headroom record: the JSONL the GPU tests append with PG_PARITY_LOG
-> one JSON summary (max errors per test, headroom = tol / max error).

    python scripts/parity_summary.py gpurun_out/parity.jsonl > profiles/r02/parity_r02.json
"""
import json
import sys


def main():
    recs = [json.loads(x) for x in open(sys.argv[1]) if x.strip()]
    vs_oracle, vs_exact = {}, []
    for r in recs:
        if r.get("test") == "error_vs_extended":
            vs_exact.append(r)
            continue
        key = f"{r['test'].split('::')[-1]} [{r['problem']}, {r['precision']}]"
        old = vs_oracle.get(key)
        if old is None or max(r["logl_rel_err"], r["grad_c17_err"]) > max(old["logl_rel_err"], old["grad_c17_err"]):
            vs_oracle[key] = {k: r[k] for k in ("N", "C", "S", "R", "logl_rel_err", "grad_c17_err",
                                                "grad_plain_rel_err_max", "tol", "headroom")}
    full = {k: v for k, v in vs_oracle.items() if "_full" in k}
    out = {"what": "CUDA path vs the fp64 oracle (C17 metric, DESIGN.md R15) for every GPU parity comparison, "
                   "and CUDA path / fp64 oracle vs the exact result of the same inputs (oracle/extended.py)",
           "min_headroom_full_size": min(v["headroom"] for v in full.values()) if full else None,
           "min_headroom_all": min(v["headroom"] for v in vs_oracle.values()),
           "full_size": full, "vs_exact_small": vs_exact, "all": vs_oracle}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
