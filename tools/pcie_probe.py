"""PCIe probe for the e2e budget: pinned H2D / D2H bandwidth of the config-3
stack and HR tiles, alone and concurrently (device-timed with CUDA events)."""
import json

import torch


def timed(fn, s, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    h_in = torch.empty(225 * 2048 * 2048, dtype=torch.uint16).pin_memory()
    d_in = torch.empty_like(h_in, device="cuda")
    h_out = torch.empty(1296 * 256 * 256 * 2, dtype=torch.float32).pin_memory()
    d_out = torch.empty_like(h_out, device="cuda")
    s = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()
    r = {}
    r["h2d_ms"] = timed(lambda: d_in.copy_(h_in, non_blocking=True), s)
    r["d2h_ms"] = timed(lambda: h_out.copy_(d_out, non_blocking=True), s)

    def both():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        d_in.copy_(h_in, non_blocking=True)
        s.wait_stream(s2)
    r["both_ms"] = timed(both, s)
    r["h2d_GBps"] = h_in.numel() * 2 / r["h2d_ms"] / 1e6
    r["d2h_GBps"] = h_out.numel() * 4 / r["d2h_ms"] / 1e6
    print(json.dumps(r))


if __name__ == "__main__":
    main()
