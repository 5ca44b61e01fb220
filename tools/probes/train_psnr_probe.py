import sys, torch, math
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from bench_configs import make
import paper_2503_01199_b200 as sb
T = sys.modules["paper_2503_01199_b200.train"]
scene, _, views, targets = make(20000, (320, 240), 3, scaled=False)
pairs = [(views[i], targets[i % len(targets)]) for i in range(3)]
orig = math.log10
def dbg(x):
    if not (x > 0): print("log10 arg", x)
    return orig(max(x, 1e-300))
T.math.log10 = dbg
for t in targets[:3]: print(t.dtype, t.shape, float(t.min()), float(t.max()))
o, ctx = sb.forward(scene, views[0])
s = torch.zeros(1, dtype=torch.float64, device="cuda")
l, g = sb.loss_and_grad(o.color, pairs[0][1], 0.2, sse_out=s)
print("sse", s.item(), ((o.color.double() - torch.as_tensor(pairs[0][1], device='cuda').double())**2).sum().item())
r = sb.train(sb.TrainConfig(epochs=1, densify=sb.DensifyConfig(budget=0)), scene, pairs)
print(r.metrics)
