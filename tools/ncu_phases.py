"""Executed instructions and stall samples of an ncu capture grouped by the
OUTERMOST physics.cuh source line of each SASS instruction's inline chain
(i.e. the line of phys_step / phys_kernel it belongs to), then by phase.

    python tools/ncu_phases.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING

CUBIN must be the same build that ran (cuobjdump -xelf all the unit's .o).
"""
import collections
import csv
import io
import re
import subprocess
import sys

PHASES = [("trunk FK", "trunk FK and velocity"), ("limb FK/RNE", "limb: FK, cdof"),
          ("CRB", "CRB mass matrix"), ("forces", "---------------- forces"),
          ("rows", "collision + constraint rows"), ("newton", "primal Newton"),
          ("diag", "diagnostics of this step"), ("euler", "semi-implicit Euler")]


def phase_starts(src):
    lines = open(src).read().splitlines()
    starts = []
    for name, marker in PHASES:
        for i, l in enumerate(lines):
            if "// ----------------" in l and marker.replace("---------------- ", "") in l:
                starts.append((i + 1, name))
                break
    return sorted(starts)


def main():
    rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    # SASS offset -> outermost physics.cuh line
    txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    fn, chain, fresh, off2line = None, [], True, {}
    for line in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'## File "([^"]+)", line (\d+)', line)
        if m:
            if fresh:
                chain = []
            fresh = False
            chain.append((m.group(1).split("/")[-1], int(m.group(2))))
            continue
        fresh = True
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", line)
        if m and fn and kname in fn:
            ph = [c for c in chain if c[0] == "physics.cuh"]
            off2line[int(m.group(1), 16)] = ph[-1] if ph else (chain[-1] if chain else None)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ai, ii, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ai], 16), float(r[ii]), float(r[si])))
        except (ValueError, IndexError):
            continue
    base = min(a for a, _, _ in data)
    import os
    starts = phase_starts(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                       "paper_2502_08844_b200", "csrc", "physics.cuh"))
    per = collections.Counter()
    smp = collections.Counter()
    ti = ts = 0
    for a, n_i, n_s in data:
        loc = off2line.get(a - base)
        if loc and loc[0] == "physics.cuh":
            name = "physics (other)"
            for ln, nm in starts:
                if loc[1] >= ln:
                    name = nm
        else:
            name = loc[0] if loc else "?"
        per[name] += n_i
        smp[name] += n_s
        ti += n_i
        ts += n_s
    for k, v in per.most_common():
        print(f"{k:20s} {100 * v / ti:5.1f}% inst  {100 * smp[k] / ts:5.1f}% samples")


if __name__ == "__main__":
    main()
