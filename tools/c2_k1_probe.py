"""K1 on the c2 snapshot (152 MiB, 21 regions), L2 flushed between calls: a launch target for ncu.
    ncu -k regex:k1_hash python tools/c2_k1_probe.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2605_03208_b200 import kc
ctx = kc.Context(0)
specs = synth.c2_specs()
vas = [ctx.alloc(s.size) for s in specs]
regions = sorted(zip(vas, [s.size for s in specs]))
C = kc.count_chunks(regions)
h = torch.zeros(C, dtype=torch.int64, device="cuda")
rarr = kc.region_array(regions)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for i in range(20):
    flush.fill_(1)
    ctx.hash(rarr, h.data_ptr())
torch.cuda.synchronize()
print("chunks", C)
