mkdir -p gpurun_out/e8
JF_GEMM_SEPI=8 timeout 600 python -m pytest tests -m gpu -x -q -k "gemm or linear or block or autograd" > gpurun_out/e8/pytest.log 2>&1
python tools/gemm_ab.py --shape mlp1 --mode exact --rounds 3 --configs "s_epi=16" "s_epi=8" > gpurun_out/e8/ab.jsonl 2>&1
python tools/gemm_ab.py --shape mlp1 --mode fast --rounds 3 --configs "s_epi=16" "s_epi=8" >> gpurun_out/e8/ab.jsonl 2>&1
python tools/gemm_ab.py --shape proj --mode exact --rounds 3 --configs "s_epi=16" "s_epi=8" >> gpurun_out/e8/ab.jsonl 2>&1
