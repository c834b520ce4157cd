"""Pinned host<->device copy bandwidth on this box (the e2e path's floor).

Times a 56 MB D2H alone, a 9 MB H2D alone, both at once on two streams, and
the D2H cut into 1/2/4/8/16 chunks -- the numbers the host-buffer forward's
chunk plan is tuned against.  Prints one JSON line.
"""
import json

import torch


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    d2h_n, h2d_n = 56_360_960, 9_175_040
    dev_o = torch.empty(d2h_n, dtype=torch.uint8, device="cuda")
    dev_i = torch.empty(h2d_n, dtype=torch.uint8, device="cuda")
    host_o = torch.empty(d2h_n, dtype=torch.uint8, pin_memory=True)
    host_i = torch.empty(h2d_n, dtype=torch.uint8, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    out["d2h_ms"] = timed(lambda: host_o.copy_(dev_o, non_blocking=True))
    out["h2d_ms"] = timed(lambda: dev_i.copy_(host_i, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            host_o.copy_(dev_o, non_blocking=True)
        with torch.cuda.stream(s2):
            dev_i.copy_(host_i, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    out["both_ms"] = timed(both)
    for k in (2, 4, 8, 16):
        step = d2h_n // k

        def chunks(k=k, step=step):
            for j in range(k):
                host_o[j * step:(j + 1) * step].copy_(dev_o[j * step:(j + 1) * step], non_blocking=True)
        out[f"d2h_{k}chunks_ms"] = timed(chunks)
    out["d2h_GBps"] = d2h_n / out["d2h_ms"] / 1e6
    out["h2d_GBps"] = h2d_n / out["h2d_ms"] / 1e6
    out["both_GBps"] = (d2h_n + h2d_n) / out["both_ms"] / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
