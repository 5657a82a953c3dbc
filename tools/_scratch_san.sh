cd $GRAFT_REPO_ROOT
bash tools/gpu_session.sh r4c sanitize tests > /dev/null 2>&1
for t in memcheck racecheck synccheck; do tail -2 gpurun_out/r4c/sanitize_$t.txt; done
tail -3 gpurun_out/r4c/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
