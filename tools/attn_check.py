"""Fused INT8-boundary attention vs a torch FP32 reference on the dequantized QKV (diagnostics)."""
import argparse, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_12422_b200 as jf
from paper_2403_12422_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=1)
ap.add_argument("--s", type=int, default=256)
ap.add_argument("--h", type=int, default=2)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--lbo", type=int, default=16384)
ap.add_argument("--sbo", type=int, default=1024)
ap.add_argument("--time", action="store_true")
ap.add_argument("--trace", action="store_true")
a = ap.parse_args()
L = _lib.lib()
L.jf_attn_set_mn_desc(a.lbo, a.sbo)
b, s, h, d = a.b, a.s, a.h, a.d
c = h * d
torch.manual_seed(0)
x = torch.randn(b * s, 3 * c, device="cuda")
qkv = jf.quantize_per_block(x)
deq = jf.dequantize(qkv).view(b, s, 3, h, d)
q, k, v = (deq[:, :, i].transpose(1, 2).float() for i in range(3))
ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(b * s, c)

oq = torch.empty(b * s, c, dtype=torch.int8, device="cuda")
os_ = torch.empty(b * s // 32, c // 32, dtype=torch.float32, device="cuda")
obf = torch.empty(b * s, c, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(b, h, s, dtype=torch.float32, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
def run():
    rc = L.jf_attn_fwd_q(qkv.values.data_ptr(), qkv.scales.data_ptr(), b, s, h, d, oq.data_ptr(), os_.data_ptr(),
                         obf.data_ptr(), lse.data_ptr(), err.data_ptr(), _lib.stream_handle())
    assert rc == 0, L.jf_last_error()
run(); torch.cuda.synchronize()
if a.trace:
    tr = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
    L.jf_attn_set_trace(tr.data_ptr()); run(); run(); torch.cuda.synchronize(); L.jf_attn_set_trace(None)
    t = tr.view(16, 64).cpu()
    t0 = t[t > 0].min().item()
    names = {2: "P:kvfree", 3: "P:conv_done", 5: "M:S_issue", 6: "M:PV_issue",
             8: "S:wait_s", 9: "S:s_full", 15: "S:s_loaded", 7: "S:max_done", 10: "S:exp_done", 11: "S:o_done", 12: "S:p_stored"}
    n = (s // 128) if True else 0
    print("tile " + " ".join(f"{v:>11s}" for v in names.values()))
    for j in range(n):
        print(f"{j:4d} " + " ".join(f"{(t[e, j].item() - t0) if t[e, j] > 0 else -1:11d}" for e in names))
    print("o_done_final", t[13, 0].item() - t0, "end", t[14, 0].item() - t0)
got = (oq.float().view(b * s // 32, 32, c // 32, 32) * os_.view(b * s // 32, 1, c // 32, 1)).view(b * s, c)
rel = ((got - ref).abs().max() / ref.abs().max()).item()
relbf = ((obf.float() - ref).abs().max() / ref.abs().max()).item()
sc = q @ k.transpose(-1, -2) / d ** 0.5
sc = sc.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device="cuda"), 1), float("-inf"))
lse_ref = torch.logsumexp(sc, -1) / 0.6931471805599453
lerr = (lse - lse_ref).abs().max().item()
print(f"b{b} s{s} h{h} d{d} lbo{a.lbo} sbo{a.sbo}: rel(codes) {rel:.3e} rel(bf16 O) {relbf:.3e} lse err {lerr:.3e} err {err.item()}")
if a.time:
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    fl = 4 * b * h * s * s * d / 2
    qb = q.to(torch.bfloat16); kb = k.to(torch.bfloat16); vb = v.to(torch.bfloat16)
    for _ in range(3): torch.nn.functional.scaled_dot_product_attention(qb, kb, vb, is_causal=True)
    e0.record()
    for _ in range(20): torch.nn.functional.scaled_dot_product_attention(qb, kb, vb, is_causal=True)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / 20
    print(f"  fused fwd {ms*1e3:.1f} us = {fl/ms/1e9:.0f} TFLOP/s; torch SDPA bf16 {ms2*1e3:.1f} us = {fl/ms2/1e9:.0f} TFLOP/s")

# ── backward ──
dattn = jf.quantize_per_block(0.1 * torch.randn(b * s, c, device="cuda"))
dO = jf.dequantize(dattn).view(b, s, h, d).transpose(1, 2)
qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
o32 = torch.nn.functional.scaled_dot_product_attention(qr, kr, vr, is_causal=True)
gq, gk, gv = torch.autograd.grad(o32, (qr, kr, vr), dO)
gref = torch.cat([g.transpose(1, 2).reshape(b * s, c) for g in (gq, gk, gv)], 1)
dq = torch.empty(b * s, 3 * c, dtype=torch.int8, device="cuda")
dqs = torch.empty(b * s // 32, 3 * c // 32, dtype=torch.float32, device="cuda")
dsum = torch.empty(b, h, s, dtype=torch.float32, device="cuda")
def runb():
    rc = L.jf_attn_bwd_q(qkv.values.data_ptr(), qkv.scales.data_ptr(), dattn.values.data_ptr(), dattn.scales.data_ptr(),
                         obf.data_ptr(), lse.data_ptr(), dsum.data_ptr(), b, s, h, d, dq.data_ptr(), dqs.data_ptr(),
                         err.data_ptr(), _lib.stream_handle())
    assert rc == 0, L.jf_last_error()
runb(); torch.cuda.synchronize()
if a.trace:
    tr = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
    L.jf_attn_set_trace(tr.data_ptr()); runb(); torch.cuda.synchronize(); L.jf_attn_set_trace(None)
    t = tr.view(16, 64).cpu()
    t0 = t[t > 0].min().item()
    names = {0: "P:cp_done", 1: "P:free", 2: "P:conv_done", 4: "M:S0_issue", 5: "M:G0_issue", 7: "C:wait_s",
             8: "C:s_full", 9: "C:p_done"}
    print("bwd (dkv CTA 0; dq kernel ran first and shares events 0-2) tile " + " ".join(f"{v:>11s}" for v in names.values()))
    for j in range(s // 128):
        print(f"{j:4d} " + " ".join(f"{(t[e, j].item() - t0) if t[e, j] > 0 else -1:11d}" for e in names))
gg = (dq.float().view(b * s // 32, 32, 3 * c // 32, 32) * dqs.view(b * s // 32, 1, 3 * c // 32, 1)).view(b * s, 3 * c)
dref = (dO * o32.detach()).sum(-1)
print(f"  bwd: dsum rel {((dsum - dref).abs().max() / dref.abs().max()).item():.3e}", end="")
for i, nm in enumerate("qkv"):
    g, r = gg[:, i * c:(i + 1) * c], gref[:, i * c:(i + 1) * c]
    print(f"  d{nm} rel {((g - r).abs().max() / r.abs().max()).item():.3e}", end="")
print(f"  err {err.item()}")
if a.time:
    for _ in range(3): runb()
    e0.record()
    for _ in range(10): runb()
    e1.record(); torch.cuda.synchronize()
    msb = e0.elapsed_time(e1) / 10
    qb.requires_grad_(True); kb.requires_grad_(True); vb.requires_grad_(True)
    ob = torch.nn.functional.scaled_dot_product_attention(qb, kb, vb, is_causal=True)
    dob = dO.to(torch.bfloat16)
    for _ in range(3): torch.autograd.grad(ob, (qb, kb, vb), dob, retain_graph=True)
    e0.record()
    for _ in range(10): torch.autograd.grad(ob, (qb, kb, vb), dob, retain_graph=True)
    e1.record(); torch.cuda.synchronize()
    msb2 = e0.elapsed_time(e1) / 10
    print(f"  fused bwd {msb*1e3:.1f} us = {2.5*fl/msb/1e9:.0f} TFLOP/s (5-GEMM count); torch SDPA bf16 bwd {msb2*1e3:.1f} us")
