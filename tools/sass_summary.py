"""Per-kernel SASS evidence for profiles/sass_summary.txt: counts of the Blackwell-native
instructions (tcgen05 MMA `UTCHMMA`, TMA `UTMALDG`/`UTMASTG`, TMEM `LDTM`/`STTM`, tcgen05 commit
`UTCBAR`) and of legacy `HMMA` (mma.sync) in every kernel of the built objects (build/*.o).

usage: python tools/sass_summary.py [build_dir] > profiles/sass_summary.txt
"""
import glob
import os
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "UTCBAR", "HMMA", "MUFU.EX2", "IMAD", "LOP3"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def short(name):
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = re.sub(r"CUtensorMap_st", "map", name)
    return name[:150]


def main():
    bdir = sys.argv[1] if len(sys.argv) > 1 else "build"
    rows = []
    for obj in sorted(glob.glob(os.path.join(bdir, "*.o"))):
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        cur, counts = None, None
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                if cur:
                    rows.append((os.path.basename(obj), cur, counts))
                cur, counts = m.group(1), dict.fromkeys(OPS, 0)
                continue
            if cur is None:
                continue
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if not m:
                continue
            op = m.group(1)
            for k in OPS:
                if op == k or op.startswith(k + "."):
                    counts[k] += 1
        if cur:
            rows.append((os.path.basename(obj), cur, counts))
    names = demangle([r[1] for r in rows])
    print("# SASS instruction counts per kernel (cuobjdump -sass of build/*.o, sm_100a)")
    print("# columns: " + " ".join(OPS))
    for (obj, _, c), n in zip(rows, names):
        if not any(c[k] for k in OPS[:7]):
            continue  # kernels with no tensor-core / TMA / TMEM / MMA instruction (elementwise)
        print(f"{obj:28s} " + " ".join(f"{c[k]:6d}" for k in OPS) + "  " + short(n))
    plain = [(o, n) for (o, _, c), n in zip(rows, names) if not any(c[k] for k in OPS[:7])]
    print(f"# {len(plain)} further kernels use CUDA cores only (elementwise / reductions / RNG):")
    for o, n in plain:
        print(f"#   {o:26s} {short(n)}")


if __name__ == "__main__":
    main()
