"""Per-kernel SASS opcode census of the built library: the instructions that
prove the Blackwell-native paths (TMA: UBLKCP / UTMALDG / UTMASTG; mbarriers:
SYNCS; tensor cores: UTC*MMA; TMEM: LDTM / STTM; packed fp32: FADD2 / FMUL2).

    python tools/sass_census.py [lib] > profiles/r02_sass_census.txt
"""
import collections
import re
import subprocess
import sys

KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "FADD2", "FFMA2", "FMUL2", "FADD",
        "DADD", "DMUL", "SHFL", "LDS", "STS", "LDG", "STG", "BAR", "LDL", "STL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return out if len(out) == len(names) else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1609_06641_b200/libchw_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = []
    cur, counts = None, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur, counts = m.group(1), collections.Counter()
            funcs.append((cur, counts))
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            counts[m.group(1)] += 1
    names = demangle([f for f, _ in funcs])
    print(f"# SASS census of {lib} ({len(funcs)} kernels); static instruction counts per kernel")
    print("# columns: " + " ".join(KEYS))
    for (f, c), nm in sorted(zip(funcs, names), key=lambda t: t[1]):
        if not any(c[k] for k in ("UBLKCP", "UTMALDG", "UTCHMMA", "FADD2", "SYNCS")):
            continue
        short = re.sub(r"\s+", " ", nm)[:150]
        print(short)
        print("    " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]))


if __name__ == "__main__":
    main()
