"""Static SASS instruction counts per kernel of the built library
(cuobjdump -sass), restricted to the mnemonics that show which sm_100a
features each kernel uses.  Writes OUT (default profiles/r02_sass_evidence.txt).

    python tools/sass_evidence.py [OUT]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2101_03403_b200", "_lib", "libcvm_b200.so")
KEEP = re.compile(r"^(UBLKCP|SYNCS|UTC\w*|LDTM|STTM|UCGABAR\w*|CGAERRBAR|MEMBAR|IMMA|DFMA|DADD|"
                  r"DMUL|LDS|STS|SHFL|BAR|FENCE)")
HEADER = """cuobjdump -sass paper_2101_03403_b200/_lib/libcvm_b200.so: static instruction counts per kernel (evidence of the sm_100a features used; tools/sass_evidence.py).
UBLKCP = cp.async.bulk (TMA bulk copy); SYNCS = mbarrier; UTCIMMA = tcgen05.mma kind::i8 (5th-gen tensor cores); UTCBAR = tcgen05.commit; LDTM = tcgen05.ld (tensor memory);
UTCCP = tcgen05.cp; UTCATOMSWS = TMEM alloc/dealloc; UCGABAR/CGAERRBAR = thread-block-cluster barrier; IMMA = legacy mma.sync int8; DFMA/DADD/DMUL = FP64 pipe;
SHFL = warp shuffle (the v4 warp FFT's lane-pair exchange); BAR = CTA / named barriers.
"""


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles",
                                                              "r02_sass_evidence.txt")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    names = dict(re.findall(r"Function : (\S+)", sass) and [])
    kern, counts = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if kern and m:
            op = m.group(1)
            if KEEP.match(op):
                counts[kern][op] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True,
                               text=True).stdout.splitlines()
    with open(out, "w") as f:
        f.write(HEADER)
        for (k, c), dn in zip(counts.items(), demangled):
            if not c:
                continue
            f.write(f"{dn[:110]}\n    " + ", ".join(f"{op} {n}" for op, n in sorted(c.items()))
                    + "\n")
    print(out, len(counts), "kernels")
    del names


if __name__ == "__main__":
    main()
