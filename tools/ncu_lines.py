"""Per-source-line totals of an ncu --set full capture (SASS source page,
instructions executed and warp-stall samples), mapped to source lines with the
-lineinfo of the same build (nvdisasm -g -c of the cubin):
  python tools/ncu_lines.py <report.ncu-rep> <kernel regex> <nvdisasm-g.txt> <mangled name> [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, dis, mangled = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# first kernel block only
i0 = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[i0:]))))
hdr = rows[0]
H = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[1:]:
    if len(r) != len(hdr) or not r[0].startswith("0x"):
        break
    data.append(r)
base = int(data[0][0], 16)
# address -> source line from nvdisasm
txt = open(dis).read()
s = txt.find(".text." + mangled)
s = txt.find("\n", s)
e = txt.find("//---------------------", s + 10)
addr2line, cur = {}, None
for l in txt[s:e].splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f'{m.group(1).split("/")[-1]}:{m.group(2)}'
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
    if m:
        addr2line[int(m.group(1), 16)] = cur
inst = collections.Counter()
stall = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
rcols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in data:
    off = int(r[0], 16) - base
    ln = addr2line.get(off, "?")
    inst[ln] += int(r[H["Instructions Executed"]] or 0)
    stall[ln] += int(r[H["Warp Stall Sampling (All Samples)"]] or 0)
    for c in rcols:
        v = int(r[H[c]] or 0)
        if v:
            reasons[ln][c[6:]] += v
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total warp instructions {ti}, stall samples {ts}")
print("| line | warp inst | % inst | stall samples | % stalls | top stalls |\n|---|---:|---:|---:|---:|---|")
for ln, v in sorted(stall.items(), key=lambda kv: -kv[1])[:top]:
    tr = ", ".join(f"{k} {n}" for k, n in reasons[ln].most_common(3))
    print(f"| {ln} | {inst[ln]} | {100 * inst[ln] / ti:.1f} | {v} | {100 * v / ts:.1f} | {tr} |")
