"""CPU-only checks: the C-ABI library loads and exports every symbol that
include/jetfire.h declares; host-side API logic (validation, analytic
counters, configs) behaves like the reference; no CPU fallback exists."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "jetfire.h")
LIB = os.path.join(ROOT, "paper_2403_12422_b200", "libjetfire.so")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(jf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    syms = _declared_symbols()
    for must in ("jf_quantize_f32", "jf_dequantize_f32", "jf_gemm_fwd", "jf_gemm_dgrad", "jf_gemm_wgrad",
                 "jf_gemm_partials", "jf_add_stats", "jf_ln_fwd", "jf_ln_bwd", "jf_gelu_fwd", "jf_gelu_bwd",
                 "jf_colsum", "jf_dropout"):
        assert must in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="libjetfire.so not built")
def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (jf_[a-z0-9_]+)", out))
    missing = [s for s in _declared_symbols() if s not in exported]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libjetfire.so not built")
def test_library_loads_and_types_without_gpu():
    import paper_2403_12422_b200 as jf
    from paper_2403_12422_b200 import _lib

    L = jf.load_library()
    assert L.jf_version() == 1
    for name in _lib.SIGNATURES:
        assert getattr(L, name).argtypes is not None
    assert L.jf_ln_bwd_workspace_bytes(64, 128) == (2 * 64 + 2 * 2 * 128) * 4
    assert L.jf_gemm_scratch_bytes(2, 64, 96, 128) == 64 * 96 + 64 * 128


def test_sm100a_only_cubin():
    lib = LIB
    if not os.path.exists(lib):
        pytest.skip("not built")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_2403_12422_b200 as jf

    with pytest.raises(jf.JetfireUnavailable):
        jf.quantize_per_block(np.ones((32, 32), np.float32))
    with pytest.raises(jf.JetfireUnavailable):
        jf.require_cuda()


def test_tileconfig_validation():
    import paper_2403_12422_b200 as jf

    assert (jf.TileConfig().b_n, jf.TileConfig().b_d) == (128, 128)
    with pytest.raises(ValueError, match="inner tile width"):
        jf.TileConfig(128, 64, 128, 32)
    with pytest.raises(ValueError, match="multiple of 16"):
        jf.TileConfig(128, 24, 128, 24)
    with pytest.raises(ValueError, match="b_n"):
        jf.TileConfig(48, 32, 128, 32)
    assert jf.TileConfig().clamped(64, 32).b_d == 32


def test_counters_closed_forms_match_reference_formula():
    from paper_2403_12422_b200.qgemm import AccessCounters, ExecMode, TileConfig, _count_call

    for n, c, d, cfg in [(256, 128, 384, TileConfig()), (160, 96, 96, TileConfig()),
                         (96, 64, 96, TileConfig(32, 32, 64, 32))]:
        k = AccessCounters()
        _count_call(k, n, c, d, cfg, ExecMode.INT8_DATA_FLOW, True)
        ls = mac = deq = q = 0
        for n0 in range(0, n, cfg.b_n):
            bn = min(cfg.b_n, n - n0)
            for d0 in range(0, d, cfg.b_d):
                bd = min(cfg.b_d, d - d0)
                ls += (bn + bd) * c + bn * bd
                mac += bn * bd * c
                deq += bn * bd * (c // 32)
                q += bn * bd
        assert k.as_tuple() == (ls, 0, mac, deq, q)
        k = AccessCounters()
        _count_call(k, n, c, d, cfg, ExecMode.QCD_EMULATION, True)
        assert k.as_tuple() == (0, ls, mac, n * d, 0)


def test_counter_log_csv():
    import paper_2403_12422_b200 as jf

    log = jf.CounterLog()
    log.add("a", 1, 1, 1, 32, jf.ExecMode.INT8_DATA_FLOW, jf.AccessCounters(1, 0, 2, 0, 0))
    log.add("b", 1, 1, 1, 32, jf.ExecMode.QCD_EMULATION, jf.AccessCounters(0, 5, 1, 3, 0))
    assert log.total().as_tuple() == (1, 5, 3, 3, 0)
    assert log.to_csv().splitlines()[0] == jf.COUNTER_CSV_HEADER


def test_block_config():
    import paper_2403_12422_b200 as jf

    assert jf.BlockConfig().head_dim == 16 and jf.BlockConfig().stats_width == 64
    assert jf.BlockConfig(c_model=96, heads=4, hidden=96).stats_width == 32
    for kw in ({"c_model": 48}, {"hidden": 100}, {"heads": 3}, {"dropout_p": 1.0}):
        with pytest.raises(ValueError):
            jf.BlockConfig(**kw)


def test_micro_mm_16():
    import paper_2403_12422_b200 as jf

    a = np.full((16, 16), 127, np.int8)
    assert (jf.micro_mm_16(a, a) == 258064).all()
    with pytest.raises(TypeError):
        jf.micro_mm_16(np.zeros((16, 16), np.int16), a)


def test_runtime_knobs():
    from paper_2403_12422_b200 import runtime

    with pytest.raises(ValueError):
        runtime.set_promotion("sloppy")
    with pytest.raises(ValueError):
        runtime.set_error_check("never")
    assert runtime.promotion_code("fast") == 1 and runtime.promotion_code("exact") == 0


@pytest.mark.parametrize("seed", [0, 10, (7, 2), 2**70 + 3, (2**64 - 1, 5)])
def test_philox_restatement_matches_numpy(seed):
    """The Philox4x64-10 stream jf_philox_keep computes == numpy's Generator(Philox).random()
    (DropoutState.generate, qnonlinear.py:190-200)."""
    from oracle import int8flow_oracle as O

    key = tuple(int(w) for w in np.random.Philox(key=seed).state["state"]["key"])
    want = np.random.Generator(np.random.Philox(key=seed)).random(37)
    assert np.array_equal(O.philox_random(key, 37), want)


def test_nvtx_ranges_wrap_ops_when_enabled(monkeypatch):
    """runtime.set_nvtx(True) wraps the public ops in named NVTX ranges;
    off by default, and the wrapped functions keep their names and signatures."""
    import inspect

    import paper_2403_12422_b200 as jf
    from paper_2403_12422_b200 import runtime

    pushed = []
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", lambda n: pushed.append(n))
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", lambda: pushed.append("pop"))

    @runtime.traced("jf.test_op")
    def op(a, b=2):
        return a + b

    assert not runtime.nvtx_enabled()
    assert op(1) == 3 and pushed == []
    runtime.set_nvtx(True)
    try:
        assert op(1, b=5) == 6 and pushed == ["jf.test_op", "pop"]
    finally:
        runtime.set_nvtx(False)
    assert jf.block_mm_forward.__name__ == "block_mm_forward"
    assert "wq" in inspect.signature(jf.block_mm_forward).parameters
