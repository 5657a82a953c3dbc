cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3p
timeout 60 python tools/attn_check.py --b 2 --s 2048 --h 32 --d 128 --trace > gpurun_out/r3p/trace.txt 2>&1
head -20 gpurun_out/r3p/trace.txt
