"""Gaps in an MP_TIMELINE dump: where the device idles between instrumented launches."""
import collections
import sys

calls, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = []
        calls.append(cur)
        continue
    n, a, b = line.split()
    cur.append((n, float(a), float(b)))
c = calls[-1]
busy = sum(b - a for _, a, b in c)
span = c[-1][2] - c[0][1]
print(f"{len(c)} launches, span {span:.2f} ms, busy {busy:.2f} ms")
gaps = collections.defaultdict(float)
big = []
for (n0, a0, b0), (n1, a1, b1) in zip(c, c[1:]):
    g = a1 - b0
    gaps[f"{n0}->{n1}"] += g
    big.append((g, n0, n1, b0))
for k, v in sorted(gaps.items(), key=lambda x: -x[1])[:12]:
    print(f"  gap {k:20s} {v:8.2f} ms")
print("largest single gaps:", [(round(g, 3), n0, n1, round(t, 2)) for g, n0, n1, t in sorted(big)[-8:]])
