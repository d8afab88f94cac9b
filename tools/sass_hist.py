"""SASS opcode histogram of the kernels in libpcvg.so (static counts; cuobjdump -sass), for the
committed evidence: DMMA / UTC*MMA / LDS / STS / UBLKCP / DFMA counts per kernel.

  python tools/sass_hist.py <regex> [<regex> ...] > profiles/r02_sass_hist.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2310_07002_b200/lib/libpcvg.so"


def main():
    pats = [re.compile(p) for p in sys.argv[1:]] or [re.compile(".")]
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if cur and m:
            funcs[cur][m.group(2)] += 1
    demangled = {}
    if funcs:
        dm = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
        demangled = dict(zip(funcs, dm))
    keys = ["DMMA", "UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UBLKCP", "UTMALDG", "LDS", "STS", "LDG", "STG", "DFMA",
            "DMUL", "DADD", "MUFU", "SYNCS", "BAR"]
    for f, cnt in funcs.items():
        name = demangled.get(f, f)
        if not any(p.search(name) for p in pats):
            continue
        total = sum(cnt.values())
        print(f"{name}\n  total {total}: " + ", ".join(f"{k} {cnt[k]}" for k in keys if cnt[k]))


if __name__ == "__main__":
    main()
