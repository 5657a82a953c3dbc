mkdir -p gpurun_out/pp
JF_GEMM_PIPE=1 timeout 600 python -m pytest tests -m gpu -x -q -k "gemm or linear or block or model" > gpurun_out/pp/pytest.log 2>&1
python tools/gemm_ab.py --shape mlp1 --mode exact --rounds 3 --configs "pipe=0" "pipe=1" > gpurun_out/pp/ab.jsonl 2>&1
python tools/gemm_ab.py --shape mlp1 --mode fast --rounds 3 --configs "pipe=0" "pipe=1" >> gpurun_out/pp/ab.jsonl 2>&1
python tools/gemm_ab.py --shape proj --mode exact --rounds 3 --configs "pipe=0" "pipe=1" >> gpurun_out/pp/ab.jsonl 2>&1
