"""Summarise a bench trace (PF_TRACE_STEPS=1 -> gpurun_out/trace_<pid>.json):
per step, the device time inside library calls, the device idle between
them, and the largest gaps / calls with what the host was doing."""
import json
import sys


def main(path):
    d = json.load(open(path))
    rows, steps = d["rows"], d["steps"]
    print("allocator before / after the timed loop:", d.get("mem"))
    bounds = [0.0] + steps
    for k in range(len(steps)):
        lo, hi = bounds[k], bounds[k + 1]
        rs = [r for r in rows if lo - 1e-6 <= r[3] < hi]
        busy = sum(r[4] - r[3] for r in rs)
        gaps = []
        prev_end, prev = lo, None
        for r in rs:
            gaps.append((r[3] - prev_end, prev[0] if prev else "-", r[0],
                         r[1], r[2]))
            prev_end, prev = r[4], r
        gaps.sort(reverse=True)
        longest = sorted(rs, key=lambda r: r[3] - r[4])[:3]
        print(f"step {k}: {hi - lo:7.2f} ms, in calls {busy:7.2f}, "
              f"{len(rs)} calls")
        for g in gaps[:3]:
            print(f"   gap {g[0]:7.2f} ms  {g[1]} -> {g[2]} "
                  f"(host issued at {g[3]:.1f}-{g[4]:.1f})")
        for r in longest:
            print(f"   call {r[4] - r[3]:7.2f} ms  {r[0]} (host {r[1]:.1f}-"
                  f"{r[2]:.1f}, device {r[3]:.1f}-{r[4]:.1f})")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)
