#!/usr/bin/env python3
"""Median / min ms per step per variant from gpurun_out/ab.log (first 2 steps dropped)."""
import re, collections, sys
d = collections.defaultdict(list)
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/ab.log'):
    m = re.match(r'(\S+) r\d (\S+) .*ms/step=\[([^\]]*)\]', l)
    if m:
        d[(m.group(1), m.group(2))] += [float(x) for x in m.group(3).split(',')[2:]]
for k, v in sorted(d.items()):
    v.sort()
    print(*k, 'median %.4f min %.4f' % (v[len(v) // 2], v[0]))
