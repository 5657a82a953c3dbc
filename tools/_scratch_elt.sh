cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3n
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 300 python tools/eltwise_bench.py > gpurun_out/r3n/elt_old.jsonl 2>&1
timeout 300 python tools/eltwise_bench.py > gpurun_out/r3n/elt_new.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3n/pytest.log 2>&1
paste <(cut -c1-60 gpurun_out/r3n/elt_old.jsonl) <(grep -o '"us": [0-9.]*, "GB/s": [0-9.]*, "frac_hbm": [0-9.]*' gpurun_out/r3n/elt_new.jsonl)
tail -3 gpurun_out/r3n/pytest.log
