import torch, time, sys
sys.path.insert(0, '.')
import paper_2410_17980_b200 as sb
dev = torch.device('cuda', 0)
B,H,L,D = 8,16,4096,128
x = [torch.randn(B,H,L,D, dtype=torch.bfloat16) .pin_memory() for _ in range(4)]
bufs = [torch.empty(B,H,L,D, dtype=torch.bfloat16, device=dev) for _ in range(4)]
def t(f, n=5):
    f(); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/n
def h2d():
    for bb, hx in zip(bufs, x): bb.copy_(hx, non_blocking=True)
print("h2d 512MiB ms", t(h2d), flush=True)
def op():
    qq,kk,vv = (z.requires_grad_(True) for z in bufs[:3])
    o = sb.stickbreaking_attention(qq,kk,vv); o.backward(bufs[3])
    for z in bufs[:3]: z.grad=None; z.requires_grad_(False)
print("autograd op ms", t(op), flush=True)
def raw():
    o, lr, fk, cache = sb.blocked_forward(bufs[0], bufs[1], bufs[2], counters=False)
    sb.blocked_backward_twophase(cache, bufs[3])
print("raw fwd+bwd ms", t(raw), flush=True)
