import sys, torch
sys.path.insert(0, '.')
from paper_2312_00407_b200 import optim, registry
from paper_2312_00407_b200.optim import Kind, OptimizerConfig
m = registry.layer_subset(registry.LLAMA_7B, 4)
shapes, n = m.shapes(), m.param_count()
p = torch.empty(n, device="cuda"); g = torch.empty(n, device="cuda")
registry.fill_params(p, shapes); registry.fill_grads(g, shapes, 1)
pb, gb = p.to(torch.bfloat16), g.to(torch.bfloat16)
del p, g
st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO), shapes)
st.apply_all(pb, gb, 5e-4)
torch.cuda.synchronize()
