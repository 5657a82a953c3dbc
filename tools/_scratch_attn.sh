cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4b
( timeout 60 python tools/attn_check.py --s 512 --h 2 --d 128
  timeout 60 python tools/attn_check.py --s 256 --h 2 --d 64
  timeout 60 python tools/attn_check.py --b 2 --s 2048 --h 32 --d 128 --time
  timeout 60 python tools/attn_check.py --b 8 --s 1024 --h 16 --d 64 --time ) > gpurun_out/r4b/attn.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_attention.py -q > gpurun_out/r4b/pytest.log 2>&1
grep "fused\|rel\|Error\|error" gpurun_out/r4b/attn.txt | head -20; tail -2 gpurun_out/r4b/pytest.log
