"""SASS census of libaurora.so: per-kernel static counts of the instructions that prove the
Blackwell paths (tcgen05.mma = UTCHMMA, TMA = UTMALDG/UTMASTG/UTMAREDG, bulk copy = UBLKCP,
tcgen05.ld = LDTM) next to legacy mma.sync (HMMA).  Writes profiles/<out>.md.

    python scripts/sass_census.py [out_name]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_06932_b200", "libaurora.so")
KEYS = ["UTCHMMA", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "LDTM", "HMMA"]


def main(out_name="r02_sass_census"):
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)[1:]
    names = [f.split("\n", 1)[0].strip() for f in funcs]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    agg = collections.OrderedDict()
    for f, d in zip(funcs, dem):
        d = d.replace("(anonymous namespace)::", "")
        short = re.sub(r"\(.*", "", d)[:80]
        c = agg.setdefault(short, dict.fromkeys(KEYS, 0))
        for k in KEYS:
            c[k] += len(re.findall(r"\b" + k + r"\b", f))
    lines = ["# SASS census of libaurora.so (cuobjdump -sass, sm_100a)", "",
             "Static instruction counts per kernel: UTCHMMA = tcgen05.mma, UTMALDG / UTMASTG / UTMAREDG = TMA tensor "
             "load / store / reduce-add, UBLKCP = 1-D bulk async copy, LDTM = tcgen05.ld, HMMA = legacy mma.sync.", "",
             "| kernel | " + " | ".join(KEYS) + " |", "|---|" + "---|" * len(KEYS)]
    for k, c in agg.items():
        if any(c.values()):
            lines.append(f"| `{k}` | " + " | ".join(str(c[x]) for x in KEYS) + " |")
    path = os.path.join(ROOT, "profiles", out_name + ".md")
    open(path, "w").write("\n".join(lines) + "\n")
    print(path)


if __name__ == "__main__":
    main(*sys.argv[1:])
