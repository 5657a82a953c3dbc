cd $GRAFT_REPO_ROOT
O=gpurun_out/r3u; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-bf16 --no-cpu --variants 0 > $O/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 12 -c 6 \
  -o $O/gemm_full -f python bench.py --steps 1 --warmup 1 --no-bf16 --no-cpu --variants 0 > $O/ncu_gemm.log 2>&1
ls -la $O
