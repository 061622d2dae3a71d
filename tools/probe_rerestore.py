"""Probe: restore -> release -> restore again at the same VAs (same process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402

ctx = kc.Context(0)
sizes = [116465322, 692060160, 4096, 65536 * 3 + 5]
vas = [ctx.alloc(s) for s in sizes]
print("vas", [hex(v) for v in vas])
image = open(synth.FIXTURE_CUBIN, "rb").read()
karg = synth.c1_kernarg(0, 0, 0, n_lists=0)
snap, cap = ctx.capture_dev(image=image, mangled="kc_fixture_walk", grid=(1, 1, 1), block=(32, 1, 1), kernarg=karg,
                            regions=[(v, s) for v, s in zip(vas, sizes)])
for v in vas:
    ctx.free(v)
for i in range(3):
    try:
        r, rep = ctx.restore_dev(snap)
        print("restore", i, "ok", [hex(x.base) for x in r.regions()])
        r.release()
    except kc.KcError as e:
        print("restore", i, "FAILED", str(e)[:300])
