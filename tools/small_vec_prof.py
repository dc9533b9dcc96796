import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2312_00407_b200 import optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig
cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
n = 4096
p = torch.randn(n, device="cuda") * 0.02
g = torch.randn(n, device="cuda") * 1e-3
st = optim.AdaLomoState(cfg, [(n,)])
for _ in range(5):
    st.apply(0, p, g, 1e-3)
torch.cuda.synchronize()
# timed, graph-captured to remove host overhead
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            st.apply(0, p, g, 1e-3)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
print("graph us per apply", a.elapsed_time(b) * 1e3 / 20)
