mkdir -p gpurun_out/nw2
cat > /tmp/t.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2403_12422_b200 as jf
jf.require_cuda()
which = sys.argv[1]
x = jf.quantize_per_block(torch.randn(256, 256, device='cuda'))
w = jf.quantize_per_block(torch.randn(256, 256, device='cuda'))
if which == "fwd": y = jf.block_mm_forward(x, w)
elif which == "dgrad": y = jf.block_mm_grad_input(x, w)
else: y = jf.block_mm_grad_weight(x, w)
torch.cuda.synchronize(); print(which, "ok")
PY
for w in fwd dgrad wgrad; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python /tmp/t.py $w >> gpurun_out/nw2/out.txt 2>&1; done
timeout 300 compute-sanitizer --tool memcheck python /tmp/t.py fwd > gpurun_out/nw2/san.txt 2>&1
