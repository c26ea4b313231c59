"""Per-kernel SASS mnemonic counts of the built sm_100a library (evidence, not product).

    python tools/sass_summary.py > profiles/r02/sass_summary.txt

Runs ``cuobjdump -sass`` on paper_2410_10503_b200/_native/libmctomo_b200.so and prints, for
every kernel of this package, the instruction count and the counts of the mnemonics that show
how the hot loops touch memory: 16-byte global gathers (LDG.E.128), shared-memory gathers
(LDS.128), 1-D TMA bulk copies (UBLKCP) with their mbarrier waits (SYNCS), packed fp32 math
(FFMA2 / FADD2), fp64 accumulation (DADD / DFMA), atomics and local-memory spills (LDL / STL).
"""

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2410_10503_b200" / "_native" / "libmctomo_b200.so"
KEYS = ["LDG.E.128", "LDG.E.64", "LDG.E", "LDS.128", "LDS", "STS", "STG.E.128", "STG.E", "UBLKCP",
        "SYNCS", "BAR.SYNC", "FFMA2", "FADD2", "FFMA", "FADD", "DADD", "DFMA", "I2FP", "ATOM",
        "RED", "LDL", "STL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                          check=True).stdout
    kernels, cur = collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
        if cur and m:
            op = m.group(1)
            kernels[cur]["_all"] += 1
            for k in KEYS:  # longest matching key first (KEYS lists specific before generic)
                if op == k or op.startswith(k + "."):
                    kernels[cur][k] += 1
                    break
    names = demangle(list(kernels))
    print(f"# {LIB.relative_to(ROOT)}: SASS mnemonic counts per kernel (cuobjdump -sass)")
    for (raw, cnt), name in zip(kernels.items(), names):
        if "cub" in raw:
            continue
        name = re.sub(r"\(anonymous namespace\)::", "", name)
        name = re.sub(r"\(.*", "", name).replace("void ", "")
        parts = ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt[k])
        print(f"{name}: {cnt['_all']} instructions; {parts}")


if __name__ == "__main__":
    sys.exit(main())
