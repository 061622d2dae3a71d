"""Probe: where does the driver place cuMemAlloc VAs, and does cuMemAddressReserve
honour a hint in a fresh process?  (hard part H1)"""
import json
import subprocess
import sys

from cuda.bindings import driver as d


def init():
    d.cuInit(0)
    err, dev = d.cuDeviceGet(0)
    err, ctx = d.cuDevicePrimaryCtxRetain(dev)
    d.cuCtxSetCurrent(ctx)


if len(sys.argv) > 1 and sys.argv[1] == "child":
    base, size = int(sys.argv[2]), int(sys.argv[3])
    init()
    err, p = d.cuMemAddressReserve(size, 2 << 20, base, 0)
    print(json.dumps({"err": int(err), "got": int(p), "want": base, "honoured": int(p) == base}))
else:
    init()
    vas = []
    for sz in [1 << 20, 64 << 20, 1 << 30]:
        err, p = d.cuMemAlloc(sz)
        vas.append(int(p))
    print("parent cuMemAlloc VAs:", [hex(v) for v in vas])
    base = vas[1] // (2 << 20) * (2 << 20)
    out = subprocess.check_output([sys.executable, __file__, "child", str(base), str(64 << 20)], text=True)
    print("fresh process reserve at parent VA:", out.strip())
    out = subprocess.check_output(["setarch", "x86_64", "-R", sys.executable, __file__, "child", str(base),
                                   str(64 << 20)], text=True)
    print("fresh process (ASLR off) reserve at parent VA:", out.strip())
