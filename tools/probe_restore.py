"""Probe (H1): in a fresh process, what does cuMemAddressReserve return for a
span captured by closure_worker capture-c1, before and after creating a kc ctx?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
d = sys.argv[1]
regs = json.load(open(os.path.join(d, "memory_regions.json")))
bases = [int(r["base"], 16) for r in regs]
print("captured bases:", [hex(b) for b in bases], "kinds:", [r["alloc_kind"] for r in regs])
from cuda.bindings import driver as drv  # noqa: E402
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
err, pctx = drv.cuDevicePrimaryCtxRetain(dev)
drv.cuCtxSetCurrent(pctx)
G = 2 << 20


def maps_near(a):
    out = []
    for ln in open("/proc/self/maps"):
        lo, hi = [int(x, 16) for x in ln.split()[0].split("-")]
        if lo <= a < hi or abs(lo - a) < (64 << 20):
            out.append(ln.strip())
    return out


for b in bases:
    sb = b // G * G
    err, p = drv.cuMemAddressReserve(G, G, sb, 0)
    print("bare ctx reserve", hex(sb), "->", int(err), hex(int(p)))
    if int(err) == 0:
        drv.cuMemAddressFree(p, G)
    print("  maps:", maps_near(sb)[:6])
err, p = drv.cuMemAddressReserve(G, G, 0, 0)
print("unhinted reserve ->", hex(int(p)))
drv.cuMemAddressFree(p, G)
from paper_2605_03208_b200 import kc  # noqa: E402
ctx = kc.Context(0)
for b in bases:
    sb = b // G * G
    err, p = drv.cuMemAddressReserve(G, G, sb, 0)
    print("after kc ctx reserve", hex(sb), "->", int(err), hex(int(p)))
    if int(err) == 0:
        drv.cuMemAddressFree(p, G)
