#!/usr/bin/env python
"""Host<->device copy rates of one B200 box: H2D alone, D2H alone, and both at
once on two streams (pinned host buffers of the e2e step's size, 537 MB), the
bound of bench.py's end-to-end number."""
import json
import sys

import torch


def main():
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 537985152
    h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        d_a.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_b, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes": nb, "h2d_ms": t1, "h2d_gbs": nb / t1 / 1e6, "d2h_ms": t2, "d2h_gbs": nb / t2 / 1e6,
                      "both_ms": t3, "both_total_gbs": 2 * nb / t3 / 1e6}))


if __name__ == "__main__":
    main()
