"""An unmodified CUDA driver-API application (no kc import): it loads the
fixture module, allocates with cuMemAlloc and launches the list walk twice
(the second in place), then writes what it saw to OUT.npz.  Used as a capture
target through CUDA_INJECTION64_PATH (paper_2605_03208_b200.cli capture)."""
import ctypes
import sys

import numpy as np
from cuda.bindings import driver as drv

sys.path.insert(0, sys.argv[2])   # the repo (synth: the fixture cubin and the c1 recipe; no kc code)
import synth  # noqa: E402


def main():
    out_path = sys.argv[1]
    assert drv.cuInit(0)[0] == drv.CUresult.CUDA_SUCCESS
    err, dev = drv.cuDeviceGet(0)
    err, pctx = drv.cuDevicePrimaryCtxRetain(dev)   # the primary context, like the CUDA runtime
    drv.cuCtxSetCurrent(pctx)
    err, mod = drv.cuModuleLoadData(open(synth.FIXTURE_CUBIN, "rb").read())
    err, fn = drv.cuModuleGetFunction(mod, b"kc_fixture_walk")
    sizes = [s.size for s in synth.C1_SPECS]
    ptrs = []
    for sz in sizes:
        err, p = drv.cuMemAlloc(sz)
        assert err == drv.CUresult.CUDA_SUCCESS, err
        ptrs.append(int(p))
    nodes, heads, out = ptrs
    init = synth.c1_fill(nodes)
    for p, arr in zip(ptrs, init):
        drv.cuMemcpyHtoD(p, arr.ctypes.data, arr.nbytes)
    types = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int)
    for mutate in (0, 1):
        err, = drv.cuLaunchKernel(fn, 32, 1, 1, 256, 1, 1, 0, 0, ((heads, out, nodes, synth.C1_N_LISTS, mutate),
                                                                   types), 0)
        assert err == drv.CUresult.CUDA_SUCCESS, err
    drv.cuCtxSynchronize()
    got = []
    for p, sz in zip(ptrs, sizes):
        h = np.zeros(sz, dtype=np.uint8)
        drv.cuMemcpyDtoH(h.ctypes.data, p, sz)
        got.append(h)
    np.savez(out_path, nodes=got[0], out=got[2], init_nodes=init[0], ptrs=np.array(ptrs, dtype=np.uint64))


if __name__ == "__main__":
    main()
