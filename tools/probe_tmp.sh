mkdir -p gpurun_out/gptl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gptl/launches.csv python bench.py --workload gpt2_medium --steps 1 --warmup 1 > gpurun_out/gptl/log 2>&1
