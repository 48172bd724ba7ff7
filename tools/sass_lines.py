"""Instruction count per source line of a cubin's kernels (nvdisasm -gi):
where the code size of a kernel comes from (instruction-cache footprint).

    python tools/sass_lines.py <cubin> [top]
"""
import collections
import re
import subprocess
import sys


def main():
    cubin, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
    fn, cur, fresh = None, None, True
    per_fn = collections.Counter()
    per_line = collections.Counter()
    for line in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'## File "([^"]+)", line (\d+)', line)
        if m:
            # the first line-info record of a block is the innermost location
            if fresh:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
            fresh = False
            continue
        fresh = True
        if fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", line):
            per_fn[fn] += 1
            if cur:
                per_line[(fn[:40], cur)] += 1
    for f, c in per_fn.most_common(8):
        print(c, f[:100])
    for (f, (src, ln)), c in per_line.most_common(top):
        print(c, src, ln, f)


if __name__ == "__main__":
    main()
