"""Lines of an ncu capture ranked by idle lane slots (32 x warp instructions -
thread instructions): where divergence / partial quads cost issue slots.

    python tools/ncu_divergence.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True, check=True).stdout
    fname, hdr, rows = None, None, []
    for row in csv.reader(io.StringIO(txt)):
        if not row:
            continue
        if row[0] == "File Name" or row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            ii = hdr.index("Instructions Executed")
            ti = hdr.index("Thread Instructions Executed")
            continue
        if hdr is None or not row[0].isdigit() or row[2] != "-":
            continue
        try:
            wi, th = float(row[ii] or 0), float(row[ti] or 0)
        except ValueError:
            continue
        if wi > 0:
            rows.append((32 * wi - th, wi, th, fname, int(row[0]), row[1][:80]))
    tw = sum(r[1] for r in rows)
    tt = sum(r[2] for r in rows)
    idle = sum(r[0] for r in rows)
    print(f"warp inst {tw:.3e}, avg active threads {tt / tw:.1f}, idle lane slots {idle:.3e}")
    for idle_l, wi, th, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * idle_l / idle:5.1f}% idle  {th / wi:5.1f} thr  {100 * wi / tw:4.1f}% inst  "
              f"{f}:{ln}  {src}")


if __name__ == "__main__":
    main()
