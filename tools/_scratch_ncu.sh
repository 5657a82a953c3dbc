cd $GRAFT_REPO_ROOT
O=gpurun_out/r4d; mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --workload gpt2_medium --steps 1 --warmup 1 --no-bf16 --no-cpu --graph 0 > $O/launches.log 2>&1
ls -la $O
