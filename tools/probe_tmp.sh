mkdir -p gpurun_out/h16d
timeout 600 python -m pytest tests -m gpu -x -q -k "gemm or partial or linear or block" > gpurun_out/h16d/pytest.log 2>&1
timeout 300 python tools/gemm_bench.py --shapes mlp1,proj --ops fwd > gpurun_out/h16d/h16.jsonl 2>&1
JF_GEMM_PROBE=6 timeout 300 python tools/gemm_bench.py --shapes mlp1 --ops fwd > gpurun_out/h16d/h16_noconv.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_h16 -s 3 -c 1 -o gpurun_out/h16d/h16_fast -f python tools/gemm_bench.py --shapes proj --ops fwd --modes fast --iters 1 > gpurun_out/h16d/ncu1.log 2>&1
