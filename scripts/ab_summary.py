#!/usr/bin/env python3
"""Summarise gpurun_out/ab.log (scripts/gpu_ab.sh): best step time per (variant, config) per round."""
import collections, re, sys
d = collections.defaultdict(list)
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.log"):
    m = re.match(r"(\S+) r\d (c\d) .*ms/step=\[([^\]]*)\]", l)
    if m:
        ms = [float(x) for x in m.group(3).split(",")][2:]
        d[(m.group(2), m.group(1))].append(min(ms))
for k, v in sorted(d.items()):
    print(k, ["%.4f" % x for x in v], "best %.4f" % min(v))
