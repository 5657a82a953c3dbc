set -u
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "gemm or partials" -m gpu -x -q > $OUT/tests_e0.log 2>&1; echo "exit $?" >> $OUT/tests_e0.log
for r in 1 2; do
for ops in int8 f16; do
  timeout 600 python tools/gemm_bench.py --shapes mlp1,proj --operands $ops > $OUT/base_${ops}_$r.jsonl 2>&1
  timeout 600 python tools/gemm_bench.py --shapes mlp1,proj --operands $ops --lib $PWD/paper_2403_12422_b200/libjetfire_e0.so > $OUT/e0_${ops}_$r.jsonl 2>&1
done; done
