cd $GRAFT_REPO_ROOT
bash tools/gpu_session.sh r3s sanitize
for t in memcheck racecheck synccheck; do tail -3 gpurun_out/r3s/sanitize_$t.txt; done
