mkdir -p gpurun_out/elp
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"add_stats|ln_fwd_kernel|gelu_fwd" -s 6 -c 3 -o gpurun_out/elp/el -f python tools/eltwise_bench.py > gpurun_out/elp/ncu.log 2>&1
