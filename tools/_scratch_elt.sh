cd $GRAFT_REPO_ROOT
O=gpurun_out/r4g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_model.py -x -q > $O/pytest.log 2>&1
timeout 900 python bench.py --workload gpt2_medium --no-cpu --no-bf16 > $O/gpt2_new.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv -k regex:ce_bf16 \
  python bench.py --workload gpt2_medium --steps 1 --warmup 1 --no-bf16 --no-cpu --graph 0 > /dev/null 2>&1
tail -2 $O/pytest.log
python -c "import json; print(json.load(open('$O/gpt2_new.json'))['value'])"
