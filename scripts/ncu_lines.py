#!/usr/bin/env python3
"""Per-source-line warp-stall samples of one kernel from an ncu --set full report.

usage: python scripts/ncu_lines.py <report.ncu-rep> <object.o> <kernel-regex> <source.cu> [top] [ncu-name-regex]
(kernel-regex matches the mangled name in the object; ncu-name-regex, default the
same, the demangled name in the report)
Maps the report's SASS rows (address order) to source lines with nvdisasm -g on
the cubin extracted from the object (built from the same source with -lineinfo).
"""
import collections, csv, os, re, subprocess, sys, tempfile

rep, obj, kre, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
nre = sys.argv[6] if len(sys.argv) > 6 else kre
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = next(f for f in os.listdir(tmp) if f.endswith(".cubin"))
sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if ".section" in l and ".text." in l and re.search(kre, l))
cur, lines = None, []
for l in sass[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(r"line (\d+)", l)
    if "//##" in l and m:
        cur = int(m.group(1))
    elif re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
        lines.append(cur)
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{nre}",
                                       "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()))
# (one block per captured launch: "Kernel Name" row, header row, instruction rows)
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
blk = rows[starts[0]:starts[1]] if len(starts) > 1 else rows[starts[0]:]
hdr, data = blk[1], [r for r in blk[2:] if len(r) == len(blk[1])]
iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
if len(data) != len(lines):
    print(f"warning: {len(data)} report rows vs {len(lines)} disassembled instructions")
agg, aex = collections.Counter(), collections.Counter()
for k, r in enumerate(data):
    ln = lines[k] if k < len(lines) else None
    agg[ln] += int(r[iss]) if r[iss].isdigit() else 0
    aex[ln] += int(r[iex]) if r[iex].isdigit() else 0
tot, totex = sum(agg.values()) or 1, sum(aex.values()) or 1
src = open(srcf).read().split("\n")
for ln, v in agg.most_common(top):
    text = src[ln - 1].strip()[:90] if ln and ln <= len(src) else "(inlined from another file)"
    print(f"line {ln}: samples {v / tot:6.1%} instr {aex[ln] / totex:6.1%}  {text}")
