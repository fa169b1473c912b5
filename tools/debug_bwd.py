import os, sys, time, subprocess, tempfile
code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
from tests.gpu_util import make_qkv
import paper_2410_17980_b200 as sb
B,H,L,d,seed = map(int, sys.argv[1:6])
q,k,v,do = make_qkv(B,H,L,d, seed=seed)
print("inputs ok", flush=True)
o, lr, st, cache = sb.blocked_forward(q,k,v); torch.cuda.synchronize(); print("fwd ok", flush=True)
if os.environ.get("SB_DEBUG_PHASES","3") != "0":
    dq,dk,dv,_ = sb.blocked_backward_twophase(cache, do); torch.cuda.synchronize(); print("bwd ok", flush=True)
'''
cfgs = [((1,1,200,64,7),"0"), ((1,1,200,64,264),"0"), ((1,3,200,64,264),"0"), ((1,1,200,64,264),"1"),
        ((1,1,192,64,7),"1"), ((1,1,200,64,7),"2"), ((1,1,320,64,7),"3"), ((1,1,136,64,7),"3")]
for cfg, ph in cfgs:
    env = dict(os.environ, SB_DEBUG_PHASES=ph)
    t = time.time()
    with tempfile.TemporaryFile("w+") as f:
        p = subprocess.Popen([sys.executable, "-c", code, *map(str, cfg)], env=env, stdout=f, stderr=subprocess.STDOUT)
        try:
            p.wait(timeout=25); status = f"rc={p.returncode}"
        except subprocess.TimeoutExpired:
            p.kill(); p.wait(); status = "TIMEOUT"
        f.seek(0); out = f.read().strip().replace("\n", " | ")[-300:]
    print(cfg, "phases", ph, f"{time.time()-t:.1f}s", status, out, flush=True)
