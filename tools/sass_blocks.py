"""Biggest straight-line SASS regions of a kernel (loop bodies): opcode mix per region.
   python tools/sass_blocks.py <mangled-kernel-name> [n]"""
import collections, re, subprocess, sys
name = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 3
txt = subprocess.run(["cuobjdump", "-sass", "-fun", name, "paper_2604_04696_b200/libgpir.so"], capture_output=True, text=True).stdout
ins = []
for line in txt.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for a, t in ins:
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, t in ins:
    if a in targets and cur:
        blocks.append(cur); cur = []
    cur.append(t)
    if "BRA" in t or "EXIT" in t:
        blocks.append(cur); cur = []
if cur: blocks.append(cur)
for b in sorted(blocks, key=len, reverse=True)[:top]:
    c = collections.Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for t in b)
    print(len(b), c.most_common(14))
