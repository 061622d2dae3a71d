"""An unmodified Triton program used as a capture TARGET (the paper's Triton
workload class) -- test workload only, not part of the
library, and it contains no library code: `paper_2605_03208_b200.cli capture`
runs it with CUDA_INJECTION64_PATH=libkc.so."""
import json

import torch
import triton
import triton.language as tl


@triton.jit
def scaled_add(x_ptr, y_ptr, out_ptr, n, alpha, BLOCK: tl.constexpr):
    pid = tl.program_id(0)
    offs = pid * BLOCK + tl.arange(0, BLOCK)
    m = offs < n
    x = tl.load(x_ptr + offs, mask=m)
    y = tl.load(y_ptr + offs, mask=m)
    tl.store(out_ptr + offs, x + alpha * y, mask=m)


def main():
    torch.manual_seed(0)
    n = 1_000_003
    x = torch.randn(n, device="cuda")
    y = torch.randn(n, device="cuda")
    out = torch.zeros(n, device="cuda")
    grid = (triton.cdiv(n, 1024),)
    for alpha in (0.5, 2.0):                  # launch #0 and launch #1
        scaled_add[grid](x, y, out, n, alpha, BLOCK=1024)
    torch.cuda.synchronize()
    expect = (x + 2.0 * y).cpu()
    print(json.dumps({"out_ok": bool(torch.equal(out.cpu(), expect)), "out_ptr": out.data_ptr(),
                      "nbytes": out.numel() * 4}))


if __name__ == "__main__":
    main()
