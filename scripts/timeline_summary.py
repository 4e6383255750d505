"""Summarises a PSG_TIMELINE Chrome trace (one rank): busy time per lane and how much of the
query the lanes overlap. Open the JSON itself in chrome://tracing or ui.perfetto.dev.

  python scripts/timeline_summary.py trace.rank0.json"""
import json
import sys


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def inter(x, y):
    i = j = 0
    tot = 0.0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if b > a:
            tot += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return tot


def main():
    ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"] if e.get("ph") == "X"]
    names = {0: "host reads", 1: "H2D copy", 2: "inflate", 3: "compute", 4: "exchange"}
    lanes = {}
    for e in ev:
        lanes.setdefault(e["tid"], []).append((e["ts"], e["ts"] + e["dur"]))
    lanes = {k: union(v) for k, v in lanes.items()}
    t0 = min(a for v in lanes.values() for a, _ in v)
    t1 = max(b for v in lanes.values() for _, b in v)
    span = t1 - t0
    print("span %.1f ms" % (span / 1000))
    for k in sorted(lanes):
        busy = sum(b - a for a, b in lanes[k])
        print("  %-11s busy %8.1f ms (%5.1f%% of the span)" % (names.get(k, k), busy / 1000, 100 * busy / span))
    for x, y in ((0, 1), (1, 3), (0, 3), (2, 3), (3, 4), (1, 4)):
        if x in lanes and y in lanes:
            print("  overlap %-11s x %-11s %8.1f ms" % (names[x], names[y], inter(lanes[x], lanes[y]) / 1000))


if __name__ == "__main__":
    main()
