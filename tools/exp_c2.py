import sys, torch
sys.path.insert(0, '.')
import phantom, paper_2012_10684_b200 as tsa
cfg = phantom.CONFIGS["c2"]
host = phantom.make_volume(cfg)
vols = [torch.from_numpy(host).cuda() for _ in range(3)]
def t(fn, n=200):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for i in range(n): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
p = tsa.make_problem(vols[0], 256, 2, 0.8)
ws = tsa.workspace_for(p, vols[0].device)
outs = [tsa.tsa_segment(v, 256, 2, 0.8) for v in vols]
print("full step      ", t(lambda i: tsa.tsa_segment(vols[i % 3], 256, 2, 0.8, out=outs[i % 3], workspace=ws)))
nol = [dict(o, labels=None) for o in outs]
print("no labels      ", t(lambda i: tsa.tsa_segment(vols[i % 3], 256, 2, 0.8, out=nol[i % 3], workspace=ws)))
print("hist (staged)  ", t(lambda i: tsa.tsa_histogram(vols[i % 3], 256)))
for hp in (2, 3, 4, 5, 6):
    print("hist_per_sm", hp, t(lambda i: tsa.tsa_segment(vols[i % 3], 256, 2, 0.8, out=outs[i % 3], workspace=ws, pipeline="compact", slab_slices=hp)))
for mt in ():
    print("mid threads", mt, t(lambda i: tsa.tsa_segment(vols[i % 3], 256, 2, 0.8, out=outs[i % 3], workspace=ws, pipeline="compact", label_lag=mt)))

# CUDA-graph replay of the step (one graph per rotating buffer)
graphs = []
s = torch.cuda.Stream()
for i in range(3):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tsa.tsa_segment(vols[i], 256, 2, 0.8, out=outs[i], workspace=ws, stream=s)
    graphs.append(g)
print("graph replay   ", t(lambda i: graphs[i % 3].replay()))
