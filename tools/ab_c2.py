"""A/B: time the c2 bench step (compact path, resident inputs rotated over
> 2x L2) with alternative library builds.  Usage: python tools/ab_c2.py a.so b.so ..."""
import subprocess
import sys

for so in sys.argv[1:] * 2:
    out = subprocess.run([sys.executable, "-c", f"""
import sys
sys.path.insert(0, '.')
import paper_2012_10684_b200 as tsa
tsa.LIB_PATH = '{so}'
import torch, phantom
cfg = phantom.CONFIGS['c2']
vol = torch.from_numpy(phantom.make_volume(cfg)).cuda()
vols = [vol] + [vol.clone() for _ in range(3)]
p = tsa.make_problem(vols[0], 256, 2, 0.8)
ws = tsa.workspace_for(p, vol.device)
outs = [dict(thresholds=torch.empty((300, 2), dtype=torch.int32, device='cuda'),
             objective=torch.empty(300, dtype=torch.float64, device='cuda'),
             histogram=torch.empty((300, 256), dtype=torch.int32, device='cuda'),
             status=torch.empty(300, dtype=torch.int32, device='cuda'),
             labels=torch.empty_like(vol)) for _ in range(4)]
s = torch.cuda.current_stream()
def step(i):
    tsa.tsa_segment(vols[i % 4], 256, 2, 0.8, out=outs[i % 4], workspace=ws, stream=s)
for i in range(20): step(i)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(2000): step(i)
e1.record(); torch.cuda.synchronize()
print('{so}', round(e0.elapsed_time(e1) / 2000 * 1e3, 2), 'us')
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:])
