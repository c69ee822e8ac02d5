import sys, torch
sys.path.insert(0, '.')
import phantom, paper_2012_10684_b200 as tsa
cfg = phantom.CONFIGS["c1"]
v = torch.from_numpy(phantom.make_volume(cfg)).cuda()
p = tsa.make_problem(v, 256, 1, 0.8)
ws = tsa.workspace_for(p, v.device)
o = tsa.tsa_segment(v, 256, 1, 0.8)
for pipe in ("compact", "fused", "staged"):
    f = lambda: tsa.tsa_segment(v, 256, 1, 0.8, out=o, workspace=ws, pipeline=pipe)
    for _ in range(20): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(500): f()
    b.record(); torch.cuda.synchronize()
    print(pipe, a.elapsed_time(b) / 500 * 1e3, "us")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa_segment(v, 256, 1, 0.8, out=o, workspace=ws, pipeline=pipe, stream=s)
    for _ in range(20): g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(500): g.replay()
    b.record(); torch.cuda.synchronize()
    print(pipe, "graph", a.elapsed_time(b) / 500 * 1e3, "us")
