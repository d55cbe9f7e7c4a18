#!/usr/bin/env python
"""Per-kernel SASS instruction summary of libtprod.so: the instructions that prove the tcgen05 /
TMEM / TMA path (UTCHMMA*, UTMALDG*, UTMASTG*, LDTM*, UTCBAR*) counted per kernel, from
`cuobjdump -sass` of the built library.  Writes profiles/sass_summary.json (committed) and is
asserted by tests/test_abi.py::test_sass_summary_matches_build.

    python scripts/sass_summary.py [--lib path] [--out profiles/sass_summary.json]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = re.compile(r"\b(UTC[A-Z0-9]*MMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG[.A-Z0-9]*|UTMAPF[.A-Z0-9]*|"
                 r"LDTM[.A-Za-z0-9]*|STTM[.A-Za-z0-9]*|UTCBAR[.A-Z0-9]*|DMMA[.A-Z0-9]*|HMMA[.A-Z0-9]*)\b")


def demangle(names):
    try:
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, timeout=60)
        out = r.stdout.splitlines()
        if len(out) == len(names):
            return out
    except Exception:
        pass
    return list(names)


def summary(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    per, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per.setdefault(cur, {})
            continue
        if cur is None:
            continue
        m = OPS.search(line)
        if m:
            op = m.group(1)
            per[cur][op] = per[cur].get(op, 0) + 1
    names = sorted(per)
    dem = demangle(names)
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    return {"library": os.path.relpath(lib, ROOT), "arch": arch,
            "kernels": {d: per[n] for n, d in zip(names, dem)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1806_07247_b200", "libtprod.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sass_summary.json"))
    a = ap.parse_args()
    s = summary(a.lib)
    with open(a.out, "w") as f:
        json.dump(s, f, indent=1, sort_keys=True)
    tot = {}
    for ops in s["kernels"].values():
        for k, v in ops.items():
            tot[k] = tot.get(k, 0) + v
    print(json.dumps({"arch": s["arch"], "kernels": len(s["kernels"]), "totals": tot}))


if __name__ == "__main__":
    main()
