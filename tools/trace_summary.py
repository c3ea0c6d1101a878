"""Summarise QRT_TRACE files: time inside each libqrt ABI entry point and the
host-side gaps between calls (where the GPU idles unless work is queued)."""
import collections
import glob
import sys

for path in sorted(glob.glob(sys.argv[1] + ".*")):
    rows = [l.split() for l in open(path)]
    rows = [(r[0], float(r[1]), float(r[2])) for r in rows if len(r) == 3]
    if not rows:
        continue
    tot = collections.Counter()
    cnt = collections.Counter()
    gaps = collections.Counter()
    prev_end, prev_name = None, None
    for name, b, e in rows:
        tot[name] += e - b
        cnt[name] += 1
        if prev_end is not None:
            gaps[f"{prev_name} -> {name}"] += max(0.0, b - prev_end)
        prev_end, prev_name = e, name
    span = rows[-1][2] - rows[0][1]
    print(f"== {path}: span {span/1e3:.1f} ms, in calls {sum(tot.values())/1e3:.1f} ms")
    for k, v in tot.most_common():
        print(f"   {k:26s} {cnt[k]:5d} calls {v/1e3:10.1f} ms")
    for k, v in gaps.most_common(6):
        print(f"   gap {k:40s} {v/1e3:10.1f} ms")
