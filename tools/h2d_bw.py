"""Pinned host->device copy bandwidth of this box (the e2e bound): one 706 MB copy (C1's
packed input per step), device-timed, plus the same split into 4 concurrent chunks on
separate streams."""
import json
import torch


def main():
    nbytes = 706478080
    h = torch.empty(nbytes // 8, dtype=torch.int64, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
        torch.cuda.synchronize()
        out["single_GBps"] = nbytes / a.elapsed_time(b) / 1e6
    ss = [torch.cuda.Stream() for _ in range(4)]
    ch = h.numel() // 4
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k, st in enumerate(ss):
            st.wait_event(a)
            with torch.cuda.stream(st):
                d[k * ch:(k + 1) * ch].copy_(h[k * ch:(k + 1) * ch], non_blocking=True)
        for st in ss:
            torch.cuda.current_stream().wait_stream(st)
        b.record()
        torch.cuda.synchronize()
        out["4stream_GBps"] = nbytes / a.elapsed_time(b) / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
