import sys, time, json, numpy as np
sys.path[:0]=['/root/repo','/root/repo/tests']
import torch, paper_1611_02274_b200 as B
from paper_1611_02274_b200 import _abi as A
from golden_cases import heat_ic, perturb
L=B.lib()
for n in (600, 700, 900, 1000):
    for wide in (0, 1):
        num=8192
        y0=perturb(heat_ic(n),0.01,42,num)
        yd=torch.from_numpy(y0).cuda(); st=torch.zeros(num*8,dtype=torch.int64,device='cuda')
        p=B.OdeProblem(A.HEAT,n,0); L.bode_set_wide(wide)
        B.int_driver_device(p,'rkc','exact',0.0,0.01,num,0,yd.data_ptr(),A.default_tol(),st.data_ptr(),0,0)
        yd.copy_(torch.from_numpy(y0)); torch.cuda.synchronize(); t=time.perf_counter()
        B.int_driver_device(p,'rkc','exact',0.0,0.01,num,0,yd.data_ptr(),A.default_tol(),st.data_ptr(),0,0)
        torch.cuda.synchronize(); dt=time.perf_counter()-t
        print(json.dumps({'n':n,'wide':wide,'sys_win_per_s':num/dt,'y0':float(yd[0])}))
L.bode_set_wide(0)
