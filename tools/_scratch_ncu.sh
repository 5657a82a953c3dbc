cd $GRAFT_REPO_ROOT
O=gpurun_out/r3z; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --workload block_h1024_s1024 --batch 8 --steps 1 --warmup 1 --no-bf16 --no-cpu --variants 0 > $O/launches.log 2>&1
ls -la $O
