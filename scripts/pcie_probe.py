"""PCIe probe (not product code): pinned host->device and device->host copy
bandwidth with 1, 2 and 4 concurrent streams, 1-D and pitched 2-D copies.

    python scripts/pcie_probe.py
"""
import json

import torch

MB = 1 << 20


def timed(fn, reps=3):
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        nbytes = fn()
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return round(best, 1)


def main():
    total = 512 * MB
    host = torch.empty(total, dtype=torch.uint8).pin_memory()
    dev = torch.empty(total, dtype=torch.uint8, device="cuda")
    out = {}
    for direction in ("h2d", "d2h"):
        for ns in (1, 2, 4, 8):
            streams = [torch.cuda.Stream() for _ in range(ns)]
            chunk = total // ns

            def go():
                cur = torch.cuda.current_stream()
                for i, s in enumerate(streams):
                    s.wait_stream(cur)
                    with torch.cuda.stream(s):
                        sl = slice(i * chunk, (i + 1) * chunk)
                        if direction == "h2d":
                            dev[sl].copy_(host[sl], non_blocking=True)
                        else:
                            host[sl].copy_(dev[sl], non_blocking=True)
                for s in streams:
                    cur.wait_stream(s)
                return total
            out[f"{direction}_{ns}streams_gbs"] = timed(go)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
