"""Per-source-line instruction and stall-sample totals from an ncu report
(--print-source cuda,sass; inlined code is attributed to its innermost line).

    python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True, check=True).stdout
    fname, hdr, per = None, None, {}
    tot_i = tot_s = 0
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            ii = hdr.index("Instructions Executed")
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or not row[0].isdigit() or row[2] != "-":
            continue  # SASS sub-rows carry an address; the line row holds the totals
        try:
            n_i, n_s = float(row[ii]), float(row[si])
        except ValueError:
            continue
        key = (fname, int(row[0]))
        per[key] = (n_i, n_s, row[1][:70])
        tot_i += n_i
        tot_s += n_s
    print(f"total instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    for (f, ln), (n_i, n_s, src) in sorted(per.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * n_i / tot_i:5.1f}% inst {100 * n_s / tot_s:5.1f}% smp  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
