mkdir -p gpurun_out/ts
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ts/pytest.log 2>&1
python tools/gemm_ab.py --shape mlp1 --mode exact --rounds 3 --configs "tma_scales=0" "tma_scales=1" > gpurun_out/ts/ab.jsonl 2>&1
python tools/gemm_ab.py --shape mlp1 --mode fast --rounds 3 --configs "tma_scales=0" "tma_scales=1" >> gpurun_out/ts/ab.jsonl 2>&1
timeout 300 python tools/gemm_bench.py --shapes proj,mlp1 > gpurun_out/ts/gemm.jsonl 2>&1
