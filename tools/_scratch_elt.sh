cd $GRAFT_REPO_ROOT
O=gpurun_out/r4h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -k "gemm or partials or linear or block" -x -q > $O/pytest.log 2>&1
for i in 1 2; do
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 900 python bench.py --workload gpt2_medium --no-cpu --no-bf16 > $O/gpt2_old_$i.json 2>/dev/null
timeout 900 python bench.py --workload gpt2_medium --no-cpu --no-bf16 > $O/gpt2_new_$i.json 2>/dev/null
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 900 python bench.py --workload block_h1024_s1024 --batch 8 --no-cpu --no-bf16 --variants 0 > $O/b1024_old_$i.json 2>/dev/null
timeout 900 python bench.py --workload block_h1024_s1024 --batch 8 --no-cpu --no-bf16 --variants 0 > $O/b1024_new_$i.json 2>/dev/null
done
JF_LIBJETFIRE=$PWD/paper_2403_12422_b200/libjetfire_old.so timeout 900 python bench.py --no-cpu --no-bf16 --variants 0 > $O/c4_old.json 2>/dev/null
timeout 900 python bench.py --no-cpu --no-bf16 --variants 0 > $O/c4_new.json 2>/dev/null
tail -1 $O/pytest.log
for f in $O/*.json; do echo "$f $(python -c "import json;d=json.load(open('$f'));print(d['value'], d.get('gemm',{}).get('tops'))")"; done
