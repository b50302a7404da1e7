#!/usr/bin/env python3
"""Op mix (ALU / FMA / LSU pipes) of the steady-state loop of a kernel's SASS.
usage: python scripts/sass_loop_mix.py <object> <mangled-kernel-name> [min_len max_len]"""
import collections, re, subprocess, sys

obj, fn = sys.argv[1], sys.argv[2]
if not fn.startswith("_Z"):  # a regex: resolve the mangled name
    names = re.findall(r"Function : (\S+)", subprocess.run(["cuobjdump", "-sass", obj],
                       capture_output=True, text=True).stdout)
    fn = next(n for n in names if re.search(fn, n))
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (300, 2000)
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for l in sass.splitlines():
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
ALU = {'IADD3', 'LOP3', 'SEL', 'ISETP', 'SHF', 'LEA', 'VIADD', 'IMNMX', 'PRMT', 'MOV', 'PLOP3', 'VIMNMX', 'IABS', 'FSEL', 'P2R', 'R2P'}
FMA = {'IMAD', 'FFMA', 'FMUL', 'FADD'}
LSU = {'LDS', 'STS', 'LDG', 'STG', 'CCTL', 'LD', 'ST', 'ATOMS', 'SHFL'}
for i, (a, t) in enumerate(ins):
    m = re.search(r'BRA (?:\S+ )?0x([0-9a-f]+)', t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr:
        continue
    body = [x for aa, x in ins if tgt <= aa <= a]
    if not (lo <= len(body) <= hi):
        continue
    ops = collections.Counter((x.split()[1] if x.startswith('@') else x.split()[0]) for x in body)
    base = collections.Counter()
    for o, c in ops.items():
        base[o.split('.')[0]] += c
    alu = sum(c for o, c in base.items() if o in ALU)
    fma = sum(c for o, c in base.items() if o in FMA)
    lsu = sum(c for o, c in base.items() if o in LSU)
    print(f"loop {hex(tgt)}-{hex(a)} len={len(body)} ALU={alu} FMA={fma} LSU={lsu} other={len(body)-alu-fma-lsu}")
    print("   ", dict(ops.most_common(25)))
