"""A/B: time c4 FULL search with alternative library builds (tools/build/*.so)."""
import os, sys, json, subprocess
for so in sys.argv[1:]:
    env = dict(os.environ, TSA_LIB=so)
    out = subprocess.run([sys.executable, "-c", f"""
import sys, os
sys.path.insert(0, '.')
import paper_2012_10684_b200 as tsa
tsa.LIB_PATH = '{so}'
import torch, phantom
cfg = phantom.CONFIGS['c4']
v = torch.from_numpy(phantom.make_volume(cfg)).cuda()
for enum in ('full', 'canonical'):
    for i in range(2): tsa.tsa_segment(v, 256, 4, 0.8, enumeration=enum)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 3 if enum == 'full' else 20
    for i in range(n): tsa.tsa_segment(v, 256, 4, 0.8, enumeration=enum)
    e1.record(); torch.cuda.synchronize()
    print('{so}', enum, e0.elapsed_time(e1)/n, 'ms')
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:])
