import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2507_21526_b200 as ta, synth
from oracle import cref
def run(hq,hkv,n,d,si,sl,last,dense,seed):
    q,k,v = synth.make_qkv(hq,hkv,n,d,seed)
    dev=torch.device('cuda'); qd,kd,vd=q.to(dev),k.to(dev),v.to(dev)
    o = ta.dense_attn_prefill(qd,kd,vd) if dense else ta.triangle_attn_prefill(qd,kd,vd,sink=si,window=sl,last_q=last)
    torch.cuda.synchronize()
    ref,_,_ = cref.attention(q,k,v,si,sl,last,dense)
    err = np.abs(o.float().cpu().double().numpy()-ref).max(axis=2)  # [h][n]
    bad = np.argwhere(err > 2e-2)
    rows = sorted(set(bad[:,1].tolist()))
    heads = sorted(set(bad[:,0].tolist()))
    print(f"n={n} hq={hq} max={err.max():.3e} nbad={len(bad)} rows[{len(rows)}]={rows[:40]} heads={heads[:40]}")
for n in [1000, 990, 1010, 1024, 960, 1100, 2000]:
    run(32,8,n,128,8,512,128,False,n)
run(32,8,1000,128,8,512,128,False,5)
run(8,2,1000,128,8,512,128,False,5)
run(4,1,1000,128,8,512,128,False,5)
