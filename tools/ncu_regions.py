"""Summarise an ncu source page (SASS) by runs of equal execution count.

usage: python tools/ncu_regions.py REPORT.ncu-rep [--dump LO HI]
Prints, per run of consecutive instructions with the same execution count,
the instruction count, stall samples and dominant opcodes -- enough to map
producer / stager / consumer regions of rollout_kernel and where their time goes.
"""
import csv
import io
import subprocess
import sys


def load(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    return hdr, rows[2:]


def main():
    hdr, data = load(sys.argv[1])
    names = [h.replace("stall_", "") for h in hdr[29:46]]
    if "--dump" in sys.argv:
        i = sys.argv.index("--dump")
        lo, hi = int(sys.argv[i + 1], 16), int(sys.argv[i + 2], 16)
        for r in data:
            ad = int(r[0], 16) & 0xFFFFF
            if lo <= ad <= hi:
                top = sorted([(int(r[29 + j]), names[j]) for j in range(17)], reverse=True)[:2]
                print(hex(ad), "%-64s" % r[1].strip()[:64], r[5], r[2],
                      [(n, v) for v, n in top if v])
        return
    prev = None
    for r in data + [None]:
        ex = int(r[5]) if r else -1
        if ex != prev:
            if prev is not None:
                top = sorted(ops.items(), key=lambda x: -x[1])[:5]
                st = sorted(stalls.items(), key=lambda x: -x[1])[:3]
                print(f"{start}-{last} ex={prev:>7} n={n:>4} samples={samp:>5} {top} {st}")
            if r is None:
                break
            prev, start, n, samp, ops, stalls = ex, r[0][-5:], 0, 0, {}, {}
        src = r[1].strip().split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "")).split(".")[0]
        n += 1
        samp += int(r[2])
        ops[op] = ops.get(op, 0) + 1
        for j in range(17):
            v = int(r[29 + j])
            if v:
                stalls[names[j]] = stalls.get(names[j], 0) + v
        last = r[0][-5:]


if __name__ == "__main__":
    main()
