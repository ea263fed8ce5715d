"""Per-stream view of an MP_TIMELINE dump (look-ahead path): panel-stream busy time by class,
the idle gaps between its launches, and how long each panel waits for the update stream."""
import collections
import sys

calls, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = []
        calls.append(cur)
        continue
    f = line.split()
    cur.append((f[0], float(f[1]), float(f[2]), int(f[3]) if len(f) > 3 else 0))
c = calls[-1]
span = max(b for _, _, b, _ in c) - c[0][1]
print(f"{len(c)} launches, span {span:.2f} ms")
streams = sorted(set(s for *_, s in c))
for sid in streams:
    r = [x for x in c if x[3] == sid]
    busy = collections.defaultdict(float)
    for n, a, b, _ in r:
        busy[n] += b - a
    gaps = sum(max(0.0, a1 - b0) for (_, _, b0, _), (_, a1, _, _) in zip(r, r[1:]))
    print(f"stream {sid}: {len(r)} launches, busy {sum(busy.values()):.2f} ms {dict((k, round(v, 2)) for k, v in busy.items())}, gaps {gaps:.2f} ms")
# panel stream: the one with leaf launches ("panel")
ps = [sid for sid in streams if any(x[0] == "panel" and x[3] == sid for x in c)]
if ps:
    r = [x for x in c if x[3] == ps[0]]
    leaf_idx = [i for i, x in enumerate(r) if x[0] == "panel"]
    per = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    starts = leaf_idx[::per]
    waits, spans, gaps_in = [], [], []
    for k, i0 in enumerate(starts):
        i1 = starts[k + 1] if k + 1 < len(starts) else len(r)
        seg = r[i0:i1]
        spans.append(seg[-1][2] - seg[0][1])
        gaps_in.append(sum(max(0.0, a1 - b0) for (_, _, b0, _), (_, a1, _, _) in zip(seg, seg[1:])))
        if k + 1 < len(starts):
            waits.append(r[i1][1] - seg[-1][2])
    print(f"panel stream: {len(starts)} panels, span/panel {1e3 * sum(spans) / len(spans):.1f} us "
          f"(in-panel gaps {1e3 * sum(gaps_in) / len(spans):.1f} us), wait before next panel "
          f"{1e3 * sum(waits) / max(1, len(waits)):.1f} us; total spans {sum(spans):.2f} ms, waits {sum(waits):.2f} ms")
    seg = r[starts[len(starts) // 2]:starts[len(starts) // 2 + 1]]
    t0 = seg[0][1]
    print("  mid panel:", [(n, round(1e3 * (a - t0), 1), round(1e3 * (b - a), 1)) for n, a, b, _ in seg])
# update-stream launches between the end of a mid panel and the start of the next one
if ps and len(streams) > 1:
    su = [sid for sid in streams if sid != ps[0] and any(x[0] == "trail" and x[3] == sid for x in c)]
    if su:
        u = [x for x in c if x[3] == su[0]]
        k = len(starts) // 2
        seg = r[starts[k]:starts[k + 1]]
        t_end = seg[-1][2]
        t_next = r[starts[k + 1]][1]
        between = [(n, round(1e3 * (a - t_end), 1), round(1e3 * (b - a), 1)) for n, a, b, _ in u if b > t_end - 0.05 and a < t_next]
        print(f"  update stream between panel {k} end and panel {k + 1} start ({1e3 * (t_next - t_end):.1f} us):", between)
if ps:
    ws = []
    for k in range(len(starts) - 1):
        seg = r[starts[k]:starts[k + 1]]
        ws.append((round(1e3 * (seg[-1][2] - seg[0][1])), round(1e3 * (r[starts[k + 1]][1] - seg[-1][2]))))
    print("  (span, wait) per panel, first 12:", ws[:12])
    print("  (span, wait) per panel, last 12:", ws[-12:])
