"""A1 allocation tracking on the GPU: CUPTI driver-API interposition of
cuMemAlloc / cuMemAllocAsync / cuMemMap (incl. torch's caching allocator),
explicit kc_alloc/kc_free feeds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cupti_interposition():
    from paper_2605_03208_b200 import build
    build.build()
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "cupti_worker.py")], capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["double_install"] == -2  # KC_ERR_STATE
    assert r["memalloc_tracked"] and r["memalloc_free_seen"]
    assert r["vmm_tracked"] and r["vmm_unmap_seen"]
    assert r["torch_segment_tracked"]
    assert r["pool_tracked"] and r["pool_free_seen"]
    assert r["untracked_after_uninstall"]


def test_explicit_tracker_feed_and_errors():
    from paper_2605_03208_b200 import build, kc
    build.build()
    ctx = kc.Context(0)
    base = 0x7F0000000000
    ctx.track(kc.KC_EV_ALLOC, base, 4096)
    ctx.track(kc.KC_EV_MAP, base + 8192, 4096, 0, kc.KC_KIND_VMM)
    with pytest.raises(kc.KcError):                  # overlap with a live region
        ctx.track(kc.KC_EV_ALLOC, base + 100, 10)
    assert [(r.base, r.size) for r in ctx.regions()] == [(base, 4096), (base + 8192, 4096)]
    ctx.track(kc.KC_EV_FREE, base + 12345)            # unknown free: warning, not fatal
    assert "untracked" in ctx.last_error()
    ctx.track(kc.KC_EV_FREE, base)
    ctx.track(kc.KC_EV_UNMAP, base + 8192)
    assert ctx.regions() == []
    a = ctx.alloc(1 << 20)                            # kc_alloc feeds the tracker itself
    assert [(r.base, r.size) for r in ctx.regions()] == [(a, 1 << 20)]
    ctx.free(a)
    assert ctx.regions() == []
    ctx.close()
