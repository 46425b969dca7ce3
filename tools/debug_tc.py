import sys, numpy as np, torch, time
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from oracle import oracle as orc
from tests import parity
cases = [(128,1,64,64,64,8,torch.bfloat16),(300,2,128,512,64,32,torch.bfloat16),(64,2,256,1024,64,16,torch.bfloat16),
         (256,1,64,128,64,8,torch.float32),(200,2,128,1024,128,16,torch.float32),(130,2,96,256,64,32,torch.float32)]
for (B,H,d_h,n_sub,d_v,k,dt) in cases:
    cfg = wl.tiny_config(B,H,d_h,n_sub,d_v,k,dt,dt, index=5)
    Q,K,V,d = wl.make_all(cfg,'cuda')
    lk = PKMLookup(H,n_sub,d_h,d_v,k,B,dt,dt)
    out, idx, w = lk.forward(Q,K,V); torch.cuda.synchronize()
    o = orc.forward(Q.cpu(),K.cpu(),V.cpu(),k)
    gi = idx.cpu().numpy()
    print((B,H,d_h,n_sub,d_v,k,str(dt)), "launches", lk.last_launch_count(), "idx equal frac", float((gi == o["idx"]).all(-1).mean()))
    try:
        _,_,rep = parity.check_forward(Q.cpu(),K.cpu(),V.cpu(),k,out,idx,w); print(rep)
    except AssertionError as e:
        print("FAIL", str(e)[:300]); print("gpu", gi[0,0,:8], "\nora", o["idx"][0,0,:8])
