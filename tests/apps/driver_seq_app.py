"""An unmodified driver-API application (no kc import) running three dependent
launches: the in-place list walk, an independent u32 axpy, and a walk that
reads the rewritten nodes.  A sequence capture target for `cli capture --count 3`."""
import ctypes
import sys

import numpy as np
from cuda.bindings import driver as drv

sys.path.insert(0, sys.argv[1])   # the repo (synth: the fixture cubin and the c1 recipe; no kc code)
import synth  # noqa: E402


def main():
    drv.cuInit(0)
    err, dev = drv.cuDeviceGet(0)
    err, pctx = drv.cuDevicePrimaryCtxRetain(dev)
    drv.cuCtxSetCurrent(pctx)
    err, mod = drv.cuModuleLoadData(open(synth.FIXTURE_CUBIN, "rb").read())
    err, walk = drv.cuModuleGetFunction(mod, b"kc_fixture_walk")
    err, axpy = drv.cuModuleGetFunction(mod, b"kc_fixture_axpy_u32")
    n_y = 100_003
    sizes = [s.size for s in synth.C1_SPECS] + [4 * n_y, 4 * n_y]
    ptrs = [int(drv.cuMemAlloc(sz)[1]) for sz in sizes]
    nodes, heads, out, x, y = ptrs
    rng = np.random.default_rng(5)
    init = list(synth.c1_fill(nodes)) + [rng.integers(0, 2**32, n_y, dtype=np.uint64).astype(np.uint32),
                                         rng.integers(0, 2**32, n_y, dtype=np.uint64).astype(np.uint32)]
    for p, arr in zip(ptrs, init):
        drv.cuMemcpyHtoD(p, arr.ctypes.data, arr.nbytes)
    wt = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int)
    drv.cuLaunchKernel(walk, 32, 1, 1, 256, 1, 1, 0, 0, ((heads, out, nodes, synth.C1_N_LISTS, 1), wt), 0)
    drv.cuLaunchKernel(axpy, (n_y + 255) // 256, 1, 1, 256, 1, 1, 0, 0,
                       ((x, y, n_y, 7), (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32)), 0)
    drv.cuLaunchKernel(walk, 32, 1, 1, 256, 1, 1, 0, 0, ((heads, out, nodes, synth.C1_N_LISTS, 0), wt), 0)
    drv.cuCtxSynchronize()


if __name__ == "__main__":
    main()
