cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3i
( timeout 60 python tools/attn_check.py --s 512 --h 2 --d 128
  timeout 60 python tools/attn_check.py --s 256 --h 2 --d 64
  timeout 60 python tools/attn_check.py --b 2 --s 2048 --h 32 --d 128 --time
  timeout 60 python tools/attn_check.py --b 8 --s 1024 --h 16 --d 64 --time ) > gpurun_out/r3i/attn.txt 2>&1
cat gpurun_out/r3i/attn.txt
