cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3q
timeout 300 ./paper_2403_12422_b200/microbench 2>&1 | head -12 > gpurun_out/r3q/mb.txt
cat gpurun_out/r3q/mb.txt
