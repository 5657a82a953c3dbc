cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3k
timeout 60 python tools/attn_check.py --b 2 --s 2048 --h 32 --d 128 --trace > gpurun_out/r3k/trace.txt 2>&1
cat gpurun_out/r3k/trace.txt | tail -22
