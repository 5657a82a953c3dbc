cd $GRAFT_REPO_ROOT
O=gpurun_out/r3y; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --workload block_h1024_s1024 --batch 8 --no-cpu > $O/bench_block_h1024.json 2> $O/bench_block_h1024.err
timeout 900 python bench.py --workload gpt2_medium --no-cpu > $O/bench_gpt2_medium.json 2> $O/bench_gpt2_medium.err
for f in $O/*.json; do echo "$f: $(python -c "import json,sys;d=json.load(open('$f'));print(d.get('value'), d.get('e2e',{}).get('value'), d.get('bf16_baseline',{}).get('int8_over_bf16'), d.get('cpu_baseline',{}).get('kind'), d.get('cpu_baseline',{}).get('value'), {k:v.get('value') for k,v in d.get('variants',{}).items()})" 2>&1 | tail -1)"; done
