#!/usr/bin/env bash
# One gpurun session: parity tests, microbenchmarks, kernel benches, bench.py,
# ncu launch list + one full capture of the top kernel.  Everything lands in
# gpurun_out/<tag>/.   usage: tools/gpu_session.sh <tag> [steps...]
#   steps: tests micro gemm eltwise bench launches ncu  (default: all)
set -u
TAG=${1:-run}
shift || true
STEPS=${*:-"tests micro gemm eltwise bench launches ncu"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
for s in $STEPS; do
  case $s in
    tests)
      JF_REPORT_DIR="$OUT" timeout 2400 python -m pytest tests -m gpu -q -rf > "$OUT/pytest_gpu.log" 2>&1
      echo "pytest exit $?" >> "$OUT/pytest_gpu.log" ;;
    parity)
      JF_REPORT_DIR="$OUT" timeout 1800 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_ref_suite.py \
        -m gpu -q -rA > "$OUT/pytest_parity.log" 2>&1
      echo "pytest exit $?" >> "$OUT/pytest_parity.log" ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py \
          > "$OUT/sanitize_$tool.txt" 2>&1
        echo "exit $?" >> "$OUT/sanitize_$tool.txt"
      done ;;
    trace)
      for m in exact fast; do for ops in int8 f16; do
        timeout 300 python tools/gemm_trace.py --shape mlp1 --mode $m --operands $ops --dump >> "$OUT/gemm_trace.txt" 2>&1
      done; done ;;
    micro)
      timeout 300 ./paper_2403_12422_b200/microbench > "$OUT/microbench.jsonl" 2>&1 ;;
    gemm)
      timeout 600 python tools/gemm_bench.py --shapes qkv,proj,mlp1,mlp2 > "$OUT/gemm_bench.jsonl" 2>&1
      timeout 600 python tools/gemm_bench.py --shapes qkv,proj,mlp1,mlp2 --operands f16 > "$OUT/gemm_bench_f16.jsonl" 2>&1 ;;
    eltwise)
      timeout 300 python tools/eltwise_bench.py > "$OUT/eltwise_bench.jsonl" 2>&1 ;;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err" ;;
    benchx)
      timeout 900 python bench.py --promotion fast --operands auto --no-cpu > "$OUT/bench_fast_auto.json" 2> "$OUT/bench_fast_auto.err"
      timeout 900 python bench.py --operands auto --no-cpu > "$OUT/bench_exact_auto.json" 2> "$OUT/bench_exact_auto.err"
      timeout 900 python bench.py --promotion fast --no-cpu --no-bf16 > "$OUT/bench_fast_int8.json" 2> "$OUT/bench_fast_int8.err" ;;
    launches)
      JF_BENCH_ELTWISE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-bf16 --no-cpu --variants 0 \
        > "$OUT/launches.log" 2>&1 ;;
    ncu)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_ -s 4 -c 1 \
        -o "$OUT/gemm_full" -f python bench.py --steps 1 --warmup 1 --no-bf16 --no-cpu \
        > "$OUT/ncu_gemm.log" 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:gelu_bwd -s 1 -c 1 \
        -o "$OUT/gelu_bwd_full" -f python bench.py --steps 1 --warmup 1 --no-bf16 --no-cpu \
        > "$OUT/ncu_gelu.log" 2>&1 ;;
  esac
done
ls -la "$OUT"
