import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2403_12422_b200 as jf
args = bench.parse(["--workload", "gpt2_medium", "--no-cpu", "--no-bf16"])
jf.require_cuda(); jf.set_error_check("deferred"); jf.runtime.set_gemm_operands(args.operands)
w = dict(bench.WORKLOADS["gpt2_medium"])
wl = bench.ModelWorkload(jf, w, args, 1, 0)
for _ in range(4): wl.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5): wl.step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(35)
