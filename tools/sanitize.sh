#!/usr/bin/env bash
# compute-sanitizer (memcheck, racecheck, synccheck) over every pipeline on a
# small c2 slab and a small k=4 / u16 problem.  Run under gpurun.
set -u
OUT=${1:-gpurun_out/sanitizer}
mkdir -p $OUT
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import phantom, paper_2012_10684_b200 as tsa
v = torch.from_numpy(phantom.make_volume(phantom.CONFIGS["c2"], nz=6, z_first=120)).cuda()
for pipe in ("compact", "fused", "staged"):
    for k in (1, 2):
        tsa.tsa_segment(v, 256, k, 0.8, pipeline=pipe)
tsa.tsa_segment(v, 256, 3, 1.0, pipeline="staged")
tsa.tsa_segment(v, 256, 4, 1.3, pipeline="staged", enumeration="full")
tsa.tsa_segment(v, 256, 2, 0.7, objective="sum_plus_product")
v16 = (v.to(torch.int32) * 13).to(torch.uint16).contiguous()
tsa.tsa_segment(v16, 4096, 2, 0.8)
# 2-D cluster kernel (staged and global-load rounds,
# 256 and 64 levels), HU path, morphology, interval DP
tsa.tsa2d_segment(v, 256, 0.8, histogram=True)
tsa.tsa2d_segment((v >> 2).contiguous(), 64, 1.0)
w = torch.from_numpy(np.random.default_rng(1).integers(0, 256, size=(2, 700, 96)).astype(np.uint8)).cuda()
tsa.tsa2d_histogram(w, 256)
h = torch.from_numpy(phantom.make_volume(phantom.CONFIGS["f2"], nz=4, z_first=120)).cuda()
tsa.tsa_hu_segment(h, 2, 0.8)
tsa.tsa_hu_preprocess(h)
tsa.tsa_morph(v[:2].contiguous(), "tophat", 10)
tsa.tsa_morph(v[:2, :37, :300].contiguous(), "open", 3)
tsa.tsa_segment(v, 256, 4, 0.8, enumeration="dp")
# round 2: k >= 3 shared-memory search (TMA staging, large-M global fallback),
# the q sweep with its single label pass, the stream and overlap pipelines,
# the tuple-sharded C-ABI call over NCCL (one rank)
tsa.tsa_segment(v, 256, 3, 0.8)
tsa.tsa_segment(v, 256, 4, 1.3)
r = torch.from_numpy(np.random.default_rng(2).integers(0, 256, size=(2, 64, 64)).astype(np.uint8)).cuda()
tsa.tsa_segment(r, 256, 3, 0.8)
tsa.tsa_segment_sweep(v, 256, 3, (0.5, 1.0, 1.5))
v5 = torch.from_numpy(phantom.make_volume(phantom.CONFIGS["c5"], nz=3, z_first=400)).cuda()
tsa.tsa_segment(v5, 4096, 2, 0.8)
tsa.tsa_segment(v5, 4096, 2, 0.8, pipeline="stream")
tsa.tsa_segment(v5, 4096, 2, 0.8, pipeline="overlap", slab_slices=2)
comm = tsa.TsaComm.nccl(1, 0, tsa.tsa_comm_unique_id())
tsa.tsa_segment_sharded(v, v.shape[0], 256, 4, 0.8, comm, mode="tuples")
comm.close()
torch.cuda.synchronize()
print("ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case.py > $OUT/$tool.log 2>&1
  echo "$tool exit=$?" | tee -a $OUT/summary.txt
  tail -3 $OUT/$tool.log >> $OUT/summary.txt
done
