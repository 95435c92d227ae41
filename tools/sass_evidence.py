"""Static SASS evidence per product kernel (cuobjdump of libmm_b200.so): counts of the mnemonics
that show how each kernel is built -- DMMA (FP64 tensor core), UTMALDG (TMA tensor loads),
UBLKCP (bulk copies), LDGSTS (cp.async), SYNCS (mbarrier), DADD/DMUL/DFMA (FP64 ALU),
LDG/STG width.  `python tools/sass_evidence.py > profiles/r01/sass_evidence.md` (no GPU needed)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1106_1347_b200", "libmm_b200.so")
KEYS = ["DMMA", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "DADD", "DMUL", "DFMA", "LDS", "LDG.E.ENL2.256",
        "STG.E.ENL2.256", "LDG", "STG", "BAR.SYNC"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + ".") or (k in ("LDG.E.ENL2.256", "STG.E.ENL2.256") and op == k):
                funcs[cur][k] += 1
                break
    demangled = {}
    try:
        names = list(funcs)
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        demangled = dict(zip(names, r.stdout.splitlines()))
    except OSError:
        pass
    print("# SASS evidence (static instruction counts per kernel, `cuobjdump -sass libmm_b200.so`)\n")
    print("Counts are instructions in the kernel's SASS (not executions).  DMMA = FP64 tensor-core MMA "
          "(`mma.sync...f64` lowers to DMMA.8x8x4 on sm_100a); UTMALDG = TMA tensor load "
          "(`cp.async.bulk.tensor`); SYNCS = mbarrier ops; LDGSTS = cp.async.\n")
    print("| kernel | " + " | ".join(KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for f, c in funcs.items():
        name = demangled.get(f, f).replace("mmk::", "").replace("void ", "")
        name = re.sub(r"\(.*$", "", name)
        if len(name) > 110:
            name = name[:110] + "…"
        print(f"| `{name}` | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")


if __name__ == "__main__":
    sys.exit(main())
