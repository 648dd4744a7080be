import torch, time
dev=torch.device("cuda:0")
for nbytes in (1_376_618, 4_194_304, 16<<20):
    h=torch.empty(nbytes//4, dtype=torch.float32).pin_memory()
    d=torch.empty(nbytes//4, dtype=torch.float32, device=dev)
    s=torch.cuda.current_stream()
    for it in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    a,b,c=[torch.cuda.Event(enable_timing=True) for _ in range(3)]
    a.record()
    for it in range(20): d.copy_(h, non_blocking=True)
    b.record()
    for it in range(20): h.copy_(d, non_blocking=True)
    c.record(); torch.cuda.synchronize()
    print(nbytes, "H2D GB/s", round(nbytes*20/a.elapsed_time(b)/1e6,1), "D2H GB/s", round(nbytes*20/b.elapsed_time(c)/1e6,1))
