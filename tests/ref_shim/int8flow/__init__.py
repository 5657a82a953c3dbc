"""TEST INFRASTRUCTURE: a numpy-facing ``int8flow`` over the B200 module.

SURVEY.md §8b's optional compat shim.  The reference's own unit suites
(``pkg/tests/test_qgemm.py``, ``test_qnonlinear.py``, ``test_qlayers.py``)
import ``int8flow.<module>`` and compare numpy arrays; with this package
first on ``sys.path`` those imports resolve here, and every hot-path call
(quantizer, dequantize, the three GEMMs, GELU, Add+stats, LayerNorm,
dropout, QuantLinear, TransformerBlock) runs on the GPU through
``paper_2403_12422_b200`` (the C ABI of libjetfire).  Inputs are uploaded,
outputs downloaded as frozen numpy arrays.

Everything OFF the hot path that the suites also import -- the FP32 helper
functions (``gelu_f32``, ``layernorm_f32``, ``compute_row_stats`` ...), the FP32
``AttentionCore``, the FP32/fake-quant twin ``ReferenceBlock`` and the
checkpoint I/O -- is taken from the UNMODIFIED reference installed in
``baseline/_ref`` (see ``_ref.py``); those are the oracles the suites compare
the GPU against.
"""
