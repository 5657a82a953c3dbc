mkdir -p gpurun_out/ab4
for i in 1 2; do
python tools/gemm_bench.py --lib paper_2403_12422_b200/libjetfire_prev.so --shapes mlp1 --ops fwd > gpurun_out/ab4/prev_$i.jsonl 2>&1
python tools/gemm_bench.py --shapes mlp1 --ops fwd > gpurun_out/ab4/new_$i.jsonl 2>&1
done
