mkdir -p gpurun_out/ab2
B="python tools/gemm_bench.py --shapes mlp1 --ops fwd"
timeout 300 $B --lib paper_2403_12422_b200/libjetfire_v1.so > gpurun_out/ab2/v1.jsonl 2>&1
timeout 300 $B --lib paper_2403_12422_b200/libjetfire_v1p.so > gpurun_out/ab2/v1p.jsonl 2>&1
JF_GEMM_EPI=8 timeout 300 $B --lib paper_2403_12422_b200/libjetfire_v1.so > gpurun_out/ab2/v1_epi8.jsonl 2>&1
JF_GEMM_ISSUERS=3 timeout 300 $B --lib paper_2403_12422_b200/libjetfire_v1.so > gpurun_out/ab2/v1_iss3.jsonl 2>&1
JF_GEMM_EPI=8 timeout 300 $B --lib paper_2403_12422_b200/libjetfire_v1p.so > gpurun_out/ab2/v1p_epi8.jsonl 2>&1
