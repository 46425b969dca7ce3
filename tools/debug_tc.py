import sys, numpy as np, torch, time
sys.path.insert(0, '.')
from paper_2602_07526_b200 import workloads as wl
from paper_2602_07526_b200.pkm import PKMLookup
from oracle import oracle as orc
from tests import parity
for (B,H,d_h,n_sub,d_v,k) in [(128,1,64,64,64,8),(300,2,128,512,64,32),(64,2,256,1024,64,16)]:
    cfg = wl.tiny_config(B,H,d_h,n_sub,d_v,k,torch.bfloat16,torch.bfloat16, index=5)
    Q,K,V,d = wl.make_all(cfg,'cuda')
    lk = PKMLookup(H,n_sub,d_h,d_v,k,B,torch.bfloat16,torch.bfloat16)
    out, idx, w = lk.forward(Q,K,V); torch.cuda.synchronize()
    o = orc.forward(Q.cpu(),K.cpu(),V.cpu(),k)
    gi = idx.cpu().numpy()
    print((B,H,d_h,n_sub,d_v,k), "launches", lk.last_launch_count(), "idx equal frac", float((gi == o["idx"]).all(-1).mean()))
    try:
        _,_,rep = parity.check_forward(Q.cpu(),K.cpu(),V.cpu(),k,out,idx,w); print(rep)
    except AssertionError as e:
        print("FAIL", str(e)[:300]); print("gpu", gi[0,0,:8], "\nora", o["idx"][0,0,:8])
