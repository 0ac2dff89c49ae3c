set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
cat > /tmp/probe_dmma.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2111_10743_b200 import _lib
lib = _lib.load()
scr = torch.zeros(148*4, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.check(lib.lb_probe_dmma(_lib.ptr(scr), 148*4, 2000, _lib.stream_handle()))
torch.cuda.synchronize()
PY
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__inst_executed.sum,launch__grid_size,sm__inst_executed_pipe_lsu.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:"dmma_peak" --csv --log-file gpurun_out/probe_ncu.csv python /tmp/probe_dmma.py > gpurun_out/probe_ncu.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:"m2l_fused|first_kernel" --launch-skip 34 --launch-count 4 --csv --log-file gpurun_out/m2l_ncu.csv python scripts/fmm_profile_c3.py > gpurun_out/m2l_ncu.log 2>&1
echo "rc=$?"
