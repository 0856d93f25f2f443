import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2411_00688_b200 as psb
x = torch.randn((512, 512), device="cuda")
st = psb.TvProxState.cold((512, 512), 50)
for _ in range(3): psb.tv_prox(x, 0.5, st)
torch.cuda.synchronize()
