import sys, torch
sys.path.insert(0, '.')
import paper_2410_17980_b200 as sb
from tests.gpu_util import make_qkv
for (B,H,L,d) in [(1,2,320,128),(1,1,256,128),(1,1,512,128),(1,1,128,64)]:
    q,k,v,do = make_qkv(B,H,L,d,seed=L+d)
    o, lr, st, c = sb.blocked_forward(q,k,v)
    a = sb.blocked_backward_twophase(c, do, store_tiles=False)
    b = sb.blocked_backward_twophase(c, do, store_tiles=True)
    torch.cuda.synchronize()
    for n,x,y in zip(('dq','dk','dv'),a[:3],b[:3]):
        diff = (x.float()-y.float()).abs()
        if diff.max() > 0:
            idx = torch.nonzero(diff[0,0] > 0)
            rows = torch.unique(idx[:,0])
            print(B,H,L,d,n,'maxdiff',diff.max().item(),'rel',(diff.max()/x.float().abs().max()).item(),'rows',rows[:10].tolist(), len(rows))
        else:
            print(B,H,L,d,n,'equal')
