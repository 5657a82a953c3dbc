mkdir -p gpurun_out/mn
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/mn/pytest.log 2>&1
timeout 300 python tools/gemm_bench.py --shapes proj,mlp1 > gpurun_out/mn/gemm.jsonl 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/mn/bench.json 2> gpurun_out/mn/bench.err
