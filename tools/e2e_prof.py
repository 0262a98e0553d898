import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_20061_b200 import pt, scenes
cfg = scenes.CONFIGS[1]
src = scenes.scene_for_config(1); blob = scenes.siren_blob(0)
W,H = cfg.width, cfg.height
host = torch.empty(W*H*3, pin_memory=True)
for it in range(6):
    torch.cuda.synchronize(); t0=time.perf_counter()
    S=pt.Scene(src); t1=time.perf_counter()
    N=pt.Nif(blob); t2=time.perf_counter()
    acc=torch.zeros(W*H*3, device='cuda'); torch.cuda.synchronize(); t3=time.perf_counter()
    pt.render_samples(S,N,W,H,0,cfg.spp,cfg.max_depth,0,acc,wave_samples=cfg.wave_samples); torch.cuda.synchronize(); t4=time.perf_counter()
    host.copy_(acc); torch.cuda.synchronize(); t5=time.perf_counter()
    S.close(); N.close(); t6=time.perf_counter()
    print(f"scene {1e3*(t1-t0):.2f} nif {1e3*(t2-t1):.2f} zero {1e3*(t3-t2):.2f} render {1e3*(t4-t3):.2f} d2h {1e3*(t5-t4):.2f} close {1e3*(t6-t5):.2f} ms")
