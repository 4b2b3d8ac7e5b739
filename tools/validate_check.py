"""Times the product validate kernel (msfft_validate_signal) on a 32-GiB
c64 batch in several process states (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2011_05698_b200 as M

def run(tag, x, reps=5):
    ms = [M.validate_signal(x) for _ in range(reps)]
    print(f"{tag:40s} kernel ms {['%.3f' % v for v in ms]}  GB/s {x.numel()*8/(np.median(ms)*1e-3)/1e9:.0f}", flush=True)

B, n = 1024, 1 << 22
x = torch.empty((B, n), dtype=torch.complex64, device="cuda")
x.real.zero_(); x.imag.zero_()
run("zeros, fresh process", x)
g = torch.Generator(device="cuda"); g.manual_seed(1)
x.copy_(torch.randn((B, n), dtype=torch.complex64, device="cuda", generator=g)) if False else None
for i in range(0, B, 64):
    x[i:i+64] = torch.randn((64, n), dtype=torch.complex64, device="cuda", generator=g)
run("randn", x)
plan = M.Plan(n, 64, M.MultiscaleConfig(), 1e-6, "complex64")
run("after Plan()", x)
seeds = np.arange(B, dtype=np.uint64)
out = (torch.empty((B, 64), dtype=torch.int64, device="cuda"), torch.empty((B, 64), dtype=torch.complex128, device="cuda"), torch.empty((B,), dtype=torch.int64, device="cuda"))
plan.execute(x, seeds, out=out, assume_valid=True)
run("after execute", x)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for av in (False, True):
    plan.execute(x, seeds, out=out, assume_valid=av)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        plan.execute(x, seeds, out=out, assume_valid=av, async_=True)
    ev[1].record(); torch.cuda.synchronize(); plan.sync()
    print("execute assume_valid", av, ev[0].elapsed_time(ev[1]) / 5, "ms/step", flush=True)
xs = x[:512]
run("half batch", xs)
x128 = torch.empty((B // 2, n), dtype=torch.complex128, device="cuda") if False else None
