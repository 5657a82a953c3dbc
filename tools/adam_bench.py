import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2403_12422_b200 as jf
from paper_2403_12422_b200 import _lib
from paper_2403_12422_b200.qtensor import empty_like_shape
jf.require_cuda(); jf.set_error_check("deferred")
L = _lib.lib()
n, c = 4096, 1024
p = torch.randn(n, c, device="cuda"); g = torch.randn(n, c, device="cuda") * 1e-3
m = torch.zeros_like(p); v = torch.zeros_like(p)
wq = empty_like_shape(n, c, p.device)
st = _lib.stream_handle()
def run():
    _lib.check(L.jf_adamw_quantize(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), n, c, 1e-4, 0.9, 0.999, 1e-8, 0.1, 0.1, 0.001, wq.values.data_ptr(), wq.scales.data_ptr(), jf.runtime.err_ptr(), st), "adamw_quantize")
for _ in range(3): run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): run()
b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 50 * 1e3
byts = n * c * 29
print(f"adamw_quantize {n}x{c}: {us:.1f} us, {byts/us/1e3:.0f} GB/s")
