"""A/B: time the f1 2-D step (c2 volume, 256 levels) with alternative library
builds.  Usage: python tools/ab_2d.py lib1.so[:cluster] lib2.so[:cluster] ..."""
import subprocess
import sys

for spec in sys.argv[1:] * 2:
    so, _, cl = spec.partition(":")
    out = subprocess.run([sys.executable, "-c", f"""
import sys
sys.path.insert(0, '.')
import paper_2012_10684_b200 as tsa
tsa.LIB_PATH = '{so}'
import torch, phantom
vol = torch.from_numpy(phantom.make_volume(phantom.CONFIGS['c2'])).cuda()
vols = [vol] + [vol.clone() for _ in range(3)]
c = {int(cl or 0)}
for i in range(3): tsa.tsa2d_segment(vols[i % 4], 256, 0.8, cluster=c)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(100): tsa.tsa2d_segment(vols[i % 4], 256, 0.8, cluster=c)
e1.record(); torch.cuda.synchronize()
print('{spec}', 'cluster', tsa.tsa2d_cluster_size(vol, 256, 0.8, c), round(e0.elapsed_time(e1) * 10, 1), 'us')
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:])
