"""Static instruction counts of the loops of one kernel (experiments only:
compare two builds before spending GPU time).

python tools/sass_loops.py file.o 'f2t_strip420It6__halfLb0' [min_len]

Disassembles the object's sm_100a cubin with inline line info (the build has
-lineinfo) and, for every backward branch (a loop) of the kernel, prints the
body length, the instructions on the hot path -- those whose source line is
not inside the rare fp16 near-zero recompute (functions named in COLD) -- and
an opcode histogram of the hot part."""
import collections
import glob
import os
import re
import subprocess
import sys
import tempfile

COLD = ("fix_tiny_row", "f2t_fix_tiny", "fix_tiny_pair", "convert_row_tiny")

obj, fun = sys.argv[1], sys.argv[2]
min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 150
src_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2308_03121_b200", "csrc")


def func_ranges(path):
    """line ranges of the functions named in COLD (brace matching)"""
    out = []
    lines = open(path).read().splitlines()
    for i, l in enumerate(lines):
        head = l + (lines[i - 1] if i else "")
        if any(re.search(r"\b%s\s*\(" % n, l) for n in COLD) and "__device__" in head:
            depth, seen = 0, False
            for j in range(i, len(lines)):
                depth += lines[j].count("{") - lines[j].count("}")
                seen = seen or "{" in lines[j]
                if seen and depth <= 0:
                    out.append((i + 1, j + 1))
                    break
    return out


cold_lines = {os.path.basename(p): func_ranges(p) for p in glob.glob(os.path.join(src_dir, "*.cu*"))}


def is_cold(stack):
    for f, ln in stack:
        for a, b in cold_lines.get(f, []):
            if a <= ln <= b:
                return True
    return False


with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
    cubin = glob.glob(os.path.join(d, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout

ins, on, stack, fresh = [], False, [], True
for line in dis.splitlines():
    if line.startswith("\t.section") or line.startswith(".section"):
        on = ".text." in line and re.search(fun, line) is not None
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', line)
    if m:
        if fresh:
            stack, fresh = [], False
        stack.append((os.path.basename(m.group(1)), int(m.group(2))))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
    if on and m:
        fresh = True
        ins.append((int(m.group(1), 16), m.group(2).strip(), is_cold(stack)))
labels = {}
for line in dis.splitlines():
    pass
addr = {a: i for i, (a, _, _) in enumerate(ins)}


def op(t):
    w = t.split()
    o = w[1] if w[0].startswith("@") else w[0]
    return o.split(".")[0]


# labels: nvdisasm -c prints `(.L_x_N) targets; resolve them from the label lines
lab = {}
cur = None
for line in dis.splitlines():
    m = re.match(r"^(\.L_x_\d+):", line.strip())
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        lab.setdefault(cur, []).append(int(m.group(1), 16))
        cur = None

seen = set()
for i, (a, t, _) in enumerate(ins):
    m = re.search(r"BRA\S*\s+.*`\((\.L_x_\d+)\)", t)
    if not m:
        continue
    cands = [x for x in lab.get(m.group(1), []) if x in addr]
    if not cands:
        continue
    tgt = min(cands, key=lambda x: abs(x - a))
    if tgt >= a:
        continue
    body = range(addr[tgt], i + 1)
    if len(body) < min_len or (tgt, a) in seen:
        continue
    seen.add((tgt, a))
    hot = [j for j in body if not ins[j][2]]
    h = collections.Counter(op(ins[j][1]) for j in hot)
    print(f"loop {tgt:#x}-{a:#x}: {len(body)} instructions, {len(hot)} hot; "
          f"STG {h['STG']} LDGSTS {h['LDGSTS']} FFMA2 {h['FFMA2']}")
    print("   ", ", ".join(f"{k} {v}" for k, v in h.most_common(26)))
