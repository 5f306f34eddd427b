import torch
x = torch.empty(4 * 1024**3 // 2, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty(1, device="cuda")
def t(f, it=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it / 1e3
s = t(lambda: torch.sum(x, dtype=torch.float32))
print(f"sum read: {x.numel()*2/s/1e9:.0f} GB/s")
xv = x.view(torch.int32)
s = t(lambda: torch.max(xv))
print(f"int max read: {xv.numel()*4/s/1e9:.0f} GB/s")
z = torch.empty_like(x)
s = t(lambda: z.copy_(x))
print(f"copy: {2*x.numel()*2/s/1e9:.0f} GB/s")
