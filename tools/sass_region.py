"""Count SASS instructions of a kernel between two source lines (nvdisasm -g).

  python tools/sass_region.py <kernel-substring> <file> <line_start> <line_end> [--print]
Builds the instruction list of the first kernel whose name contains the
substring and reports the address span from the first instruction tagged
with line_start to the last tagged with line_end (first occurrence span)."""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    kname, fname, l0, l1 = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    so = os.path.join(ROOT, "paper_2302_05176_b200", "libgmsketch_b200.so")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = txt.splitlines()
    start = None
    for i, ln in enumerate(lines):
        if ln.startswith(".text.") and kname in ln:
            start = i
            break
    assert start is not None, "kernel not found"
    cur = None
    ins = []
    for ln in lines[start + 1:]:
        if ln.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), cur, m.group(2)))
    a0 = next(a for a, c, _ in ins if c and c[0] == fname and c[1] == l0)
    a1 = next(a for a, c, _ in ins if c and c[0] == fname and c[1] == l1 and a > a0)
    span = [x for x in ins if a0 <= x[0] <= a1]
    print(f"{len(span)} instructions from 0x{a0:x} to 0x{a1:x}")
    if "--print" in sys.argv:
        for a, c, t in span:
            print(f"0x{a:05x} {c[0][:10] if c else ''}:{c[1] if c else ''} {t}")


if __name__ == "__main__":
    main()
