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
    err = np.abs(o.float().cpu().double().numpy()-ref).max(axis=2)
    bad = np.argwhere(err > 2e-2)
    print(f"n={n} hq={hq} d={d} dense={dense} max={err.max():.3e} nbad={len(bad)} rows={sorted(set(bad[:,1].tolist()))[:20]} heads={sorted(set(bad[:,0].tolist()))[:10]}", flush=True)
import os
CASES=[(1,1,512,64,4,64,64,True),(1,1,512,64,4,64,64,False),(8,2,900,64,0,1,1,True),(32,8,1000,128,8,512,128,False),(32,8,4097,128,8,512,128,False)]
if os.environ.get('CASE'): CASES=[CASES[int(os.environ['CASE'])]]
for args in CASES:
    run(*args, seed=5)
