"""SASS instruction mix per kernel of libspmoe.so (cuobjdump -sass): the
tcgen05 / TMA / TMEM evidence (UTCHMMA = tcgen05.mma, UTMALDG = TMA tensor
load, UBLKCP = cp.async.bulk, LDTM = tcgen05.ld, UTCBAR = tcgen05.commit,
SYNCS = mbarrier ops) next to the CUDA-core kernels' FFMA / LDG counts.

python tools/sass_summary.py [--lib paper_2510_10302_b200/libspmoe.so] > profiles/r2_sass_summary.txt
"""

from __future__ import annotations

import argparse
import collections
import re
import subprocess

KEYS = ["UTCHMMA", "UTMALDG", "UBLKCP", "LDTM", "UTCBAR", "SYNCS", "ELECT", "LDG", "STG", "LDS", "STS", "FFMA",
        "SHFL", "BAR"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="paper_2510_10302_b200/libspmoe.so")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    stats: dict[str, collections.Counter] = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            stats[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            stats[cur]["total"] += 1
            if m.group(1) in KEYS:
                stats[cur][m.group(1)] += 1
    names = subprocess.run(["c++filt"], input="\n".join(stats), capture_output=True, text=True).stdout.splitlines()
    print(f"# cuobjdump -sass {a.lib}  ({', '.join(arch)}); static instruction counts per kernel")
    print("kernel," + ",".join(["total"] + KEYS))
    for (mangled, c), name in zip(stats.items(), names):
        short = re.sub(r"\(anonymous namespace\)::", "", name)
        short = re.sub(r"^void ", "", short).split("(")[0]
        print(f"{short}," + ",".join(str(c.get(k, 0)) for k in ["total"] + KEYS))


if __name__ == "__main__":
    main()
