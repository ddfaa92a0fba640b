"""SASS evidence for the shipped kernels (cuobjdump -sass of libbf16x.so): per kernel, counts of
the Blackwell tensor-core / TMA / TMEM instructions that prove the path --
UTCHMMA / UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), UTMALDG (TMA tensor load),
UTMAPF (TMA descriptor prefetch), LDTM (tcgen05.ld), and local-memory spills (LDL / STL).
Writes profiles/r08/sass_counts.txt."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMAPF", "LDTM", "STTM", "SYNCS", "LDL", "STL"]


def main():
    lib = os.path.join(ROOT, "paper_1904_06376_b200", "libbf16x.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    counts[cur][o] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    lines = ["kernel | " + " | ".join(OPS)]
    for (name, c), dn in zip(counts.items(), demangle):
        if not any(c[o] for o in OPS):
            continue
        short = re.sub(r"\(.*", "", dn).replace("bf16x::", "")
        lines.append(f"{short} | " + " | ".join(str(c[o]) for o in OPS))
    out = "\n".join(lines)
    print(out)
    os.makedirs(os.path.join(ROOT, "profiles", "r08"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r08", "sass_counts.txt"), "w") as f:
        f.write("# cuobjdump -sass paper_1904_06376_b200/libbf16x.so (tools/sass_counts.py)\n" + out + "\n")


if __name__ == "__main__":
    sys.exit(main())
