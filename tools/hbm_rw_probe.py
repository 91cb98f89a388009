import torch
x = torch.ones(2 * 1024**3, dtype=torch.int32, device="cuda")  # 8 GiB
y = torch.empty(1024**3, dtype=torch.int32, device="cuda")
def t(fn, nbytes, name):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {ms:.3f} ms {nbytes/ms/1e6:.0f} GB/s", flush=True)
t(lambda: x.sum(dtype=torch.int64), x.numel()*4, "read-only sum 8 GiB")
t(lambda: torch.amax(x.view(-1, 1024), dim=1), x.numel()*4, "read amax rows")
t(lambda: y.fill_(3), y.numel()*4, "write-only fill 4 GiB")
t(lambda: y.copy_(x[:y.numel()]), y.numel()*8, "copy 4 GiB (r+w)")
