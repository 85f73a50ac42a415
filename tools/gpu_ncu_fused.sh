cat > /tmp/iir_only.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine
fs, C, dur = 48000, 32, 30.0
N = int(dur * fs)
w = wp.white_noise(dur, C, fs, seed=42); x = w.tensor(); y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
plan = engine.plan_for(wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000)]).bind(fs).stages, device=0)
nb = plan.workspace_bytes(C, N); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
for _ in range(3): plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
PY
WP_CHAIN_IMPL=cuda timeout 600 ncu --set full --import-source on -k regex:fused_chain -s 2 -c 1 -o gpurun_out/prof_fused_iir python /tmp/iir_only.py > gpurun_out/ncu_fused.log 2>&1
tail -2 gpurun_out/ncu_fused.log
