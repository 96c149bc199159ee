"""A/B timing of the fused L1 + SSIM loss (k_ssim_fwd + k_ssim_adj + finalize) at c3
resolution (1920 x 1080 x 3), one stream, CUDA events.  Usage:
    python profiles/loss_exp.py [path/to/libtgs variant .so ...]
Each library is timed in a fresh subprocess (the ctypes handle is per process)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(lib):
    import torch
    from paper_2501_14534_b200 import _lib
    if lib:
        _lib.LIB_PATH = os.path.abspath(lib)
    from paper_2501_14534_b200 import loss as L
    g = torch.Generator(device="cuda").manual_seed(0)
    img = torch.rand((1080, 1920, 3), device="cuda", generator=g)
    tgt = torch.rand((1080, 1920, 3), device="cuda", generator=g)
    d = torch.empty_like(img)
    terms = torch.zeros(2, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(10):
        L.l1_ssim_async(img, tgt, 0.2, d, terms)
    ts = []
    for _ in range(50):
        flush.zero_()  # cold L2 like the training step (other views' kernels in between)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.l1_ssim_async(img, tgt, 0.2, d, terms)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    chk = float(d.double().abs().sum()), terms.tolist()
    print(f"{lib or 'libtgs.so'}: median {ts[len(ts) // 2]:.1f} us  min {ts[0]:.1f} us  check {chk}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        run(sys.argv[2] if len(sys.argv) > 2 else "")
    else:
        for lib in [""] + sys.argv[1:]:
            subprocess.run([sys.executable, __file__, "--one", lib], check=True)
