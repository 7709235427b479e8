import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_09983_b200 import abi
from paper_2603_09983_b200.configs import CONFIGS, SYNTH_STD
w = CONFIGS['tiny'].with_(cache_ratio=float(sys.argv[1]))
L,N,k,g,d,ffn,T = w.n_layers,w.n_experts,w.top_k,w.gamma,w.d_model,w.d_ffn,w.tokens
cfg = abi.default_config(n_layers=L, n_experts=N, top_k=k, gamma=g, cache_ratio=w.cache_ratio)
ctx = abi.Context(0, w.model_desc(), cfg); ctx.host_arena(9); ctx.fill_synthetic(3, SYNTH_STD); ctx.finalize()
synth = abi.TraceSynth(cfg)
S=200
lh = torch.empty((S,L,T,N),dtype=torch.float64).pin_memory()
acc=[synth.next(lh[s].numpy())[1] for s in range(S)]
hh = torch.randn((S,T,d)).to(torch.bfloat16).pin_memory()
ho = torch.empty((T,d),dtype=torch.bfloat16).pin_memory()
ld, hd = lh.cuda(), hh.cuda(); hod=torch.empty((T,d),dtype=torch.bfloat16,device='cuda')
ln = [lh[s].numpy() for s in range(S)]; hn=[hh[s].view(torch.int16).numpy() for s in range(S)]; hon=ho.view(torch.int16).numpy()
for i in range(20): ctx.step(ln[i], hn[i], acc[i], hon)
def tm(f, n=150):
    torch.cuda.synchronize(); t=time.perf_counter()
    for i in range(n): f(20+i)
    torch.cuda.synchronize(); return (time.perf_counter()-t)/n*1e6
print('host step (prebuilt views) us', tm(lambda s: ctx.step(ln[s], hn[s], acc[s], hon)))
print('host step (views per step) us', tm(lambda s: ctx.step(lh[s].numpy(), hh[s].view(torch.int16).numpy(), acc[s], hon)))
print('device step us', tm(lambda s: ctx.step_device(ld[s], hd[s], acc[s], hod)))
ctx.set_timing(True)
r=[ctx.step_device(ld[20+i], hd[20+i], acc[20+i], hod)[0] for i in range(50)]
print('gpu_ms_total', np.mean([x.gpu_ms_total for x in r]), 'ffn', np.mean([x.gpu_ms_ffn for x in r]), 'launches', r[0].kernel_launches)
