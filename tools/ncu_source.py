"""Per-instruction view of an ncu report's SASS source page: the instructions
with the most excess shared-memory wavefronts, the top stall sites, and an
opcode histogram weighted by executed instructions.

    python tools/ncu_source.py gpurun_out/x.ncu-rep [--top 15]
"""
import collections
import csv
import io
import subprocess
import sys


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    return rows[0], rows[1:]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
    hdr, rows = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    ex = [(f(r[ix["L1 Wavefronts Shared Excessive"]]), r[ix["Address"]], r[ix["Source"]]) for r in rows]
    ex.sort(reverse=True)
    print("== excess shared wavefronts")
    for e in ex[:top]:
        if e[0] > 0:
            print(f"  {e[0]:>12.0f}  {e[1]}  {e[2][:90]}")
    st = [(f(r[ix["Warp Stall Sampling (All Samples)"]]), r[ix["Address"]], r[ix["Source"]]) for r in rows]
    st.sort(reverse=True)
    tot = sum(s[0] for s in st) or 1
    print("== stall samples")
    for s in st[:top]:
        print(f"  {100 * s[0] / tot:5.1f}%  {s[1]}  {s[2][:90]}")
    hist = collections.Counter()
    for r in rows:
        op = r[ix["Source"]].split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else "")
        hist[o.split(".")[0]] += f(r[ix["Instructions Executed"]])
    n = sum(hist.values()) or 1
    print("== executed warp instructions by opcode")
    for o, c in hist.most_common(25):
        print(f"  {o:10s} {c:14.0f}  {100 * c / n:5.1f}%")


if __name__ == "__main__":
    main()
