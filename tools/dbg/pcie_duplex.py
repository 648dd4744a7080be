"""PCIe duplex probe: D2H of the 4.19 MB DLRM-small result and H2D of its 1.38 MB inputs, each
alone and both at once on two streams (the e2e serving loop's traffic), pinned host memory."""
import json, torch
dev = torch.device("cuda:0")
n_out, n_in, K = 4_194_304, 1_376_618, 50
ho = [torch.empty(n_out // 4).pin_memory() for _ in range(2)]
hi = [torch.empty(n_in // 4).pin_memory() for _ in range(2)]
do = torch.empty(n_out // 4, device=dev)
di = [torch.empty(n_in // 4, device=dev) for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(d2h, h2d):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_event(a); s2.wait_event(a)
    for k in range(K):
        if d2h:
            with torch.cuda.stream(s1): ho[k & 1].copy_(do, non_blocking=True)
        if h2d:
            with torch.cuda.stream(s2): di[k & 1].copy_(hi[k & 1], non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / K
for _ in range(2): run(True, True)
out = {"d2h_only_us": run(True, False), "h2d_only_us": run(False, True), "both_us": run(True, True)}
out["d2h_only_gbs"] = n_out / out["d2h_only_us"] / 1e3
out["h2d_only_gbs"] = n_in / out["h2d_only_us"] / 1e3
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
