cd $GRAFT_REPO_ROOT
O=gpurun_out/r3x; mkdir -p $O
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 300 python tools/eltwise_bench.py > $O/elt_old.jsonl 2>&1
timeout 300 python tools/eltwise_bench.py > $O/elt_new.jsonl 2>&1
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 300 python tools/eltwise_bench.py > $O/elt_old2.jsonl 2>&1
timeout 300 python tools/eltwise_bench.py > $O/elt_new2.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not ref_suite" > $O/pytest.log 2>&1
paste <(cut -c1-30 $O/elt_old.jsonl) <(grep -o '"us": [0-9.]*' $O/elt_old.jsonl) <(grep -o '"us": [0-9.]*' $O/elt_old2.jsonl) <(grep -o '"us": [0-9.]*' $O/elt_new.jsonl) <(grep -o '"us": [0-9.]*' $O/elt_new2.jsonl)
tail -1 $O/pytest.log
