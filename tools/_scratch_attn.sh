cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4a
( timeout 60 python tools/attn_check.py --s 512 --h 2 --d 128
  timeout 60 python tools/attn_check.py --s 256 --h 2 --d 64
  timeout 60 python tools/attn_check.py --b 2 --s 2048 --h 32 --d 128 --time --trace
  timeout 60 python tools/attn_check.py --b 8 --s 1024 --h 16 --d 64 --time ) > gpurun_out/r4a/attn.txt 2>&1
grep -v "^ *[0-9]* *[0-9-]* " gpurun_out/r4a/attn.txt | head -30; grep -A20 "^tile" gpurun_out/r4a/attn.txt | head -18
