"""bench.py helpers that need no GPU: the roofline object and the DP payload shapes."""

import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_roofline_fields():
    r = bench.roofline(480.0, "exact", clocks_mhz=1965.0, operands="int8")
    for k in ("kernel", "bound", "achieved", "peak", "unit", "frac", "traffic", "promotion_bound"):
        assert k in r, k
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert abs(r["frac"] - 480.0 / bench.INT8_PEAK_TOPS) < 1e-4
    pb = r["promotion_bound"]
    assert abs(pb["value"] - 128.0 / 3 * 64 * 148 * 1965e6 / 1e12) < 0.1
    assert "gemm_tc_kernel<OP_I8>" in r["kernel"] and "measured_peak" in r
    assert "gemm_tc_kernel<OP_F16>" in bench.roofline(480.0, "exact", operands="auto")["kernel"]


def test_grad_shapes_block_and_linear():
    def lin(d, c, bias=True):
        return types.SimpleNamespace(master_weight=types.SimpleNamespace(shape=(d, c)),
                                     bias=types.SimpleNamespace(shape=(d,)) if bias else None)

    ln = types.SimpleNamespace(gamma=types.SimpleNamespace(shape=(64,)), beta=types.SimpleNamespace(shape=(64,)))
    blk = types.SimpleNamespace(qkv=lin(192, 64), proj=lin(64, 64), mlp1=lin(256, 64), mlp2=lin(64, 256, False),
                                ln1=ln, ln2=ln)
    s = bench.grad_shapes(types.SimpleNamespace(blk=blk))
    assert s["qkv.w"] == (192, 64) and s["mlp1.b"] == (256,) and "mlp2.b" not in s
    assert s["ln2.beta"] == (64,) and len(s) == 11
    assert bench.grad_shapes(types.SimpleNamespace(lin=lin(8, 4))) == {"w": (8, 4), "b": (8,)}


def test_workloads_and_parse():
    a = bench.parse([])
    assert a.workload == "block_h4096_s2048" and a.operands == "int8" and a.overlap_wgrad == 1
    for name in ("block_h4096_s2048", "block_h1024_s1024", "gpt2_medium", "gpt2_large", "linear_n4096"):
        assert name in bench.WORKLOADS
