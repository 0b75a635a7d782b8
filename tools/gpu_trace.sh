JTFS_NVCC_EXTRA=-DJTFS_TC_TRACE python -c "
import sys; sys.path.insert(0,'.')
from paper_2602_11896_b200 import build as b; b.build(force=True)" > gpurun_out/trace_build.log 2>&1
for k in 18 34; do
  JTFS_TRACE_K=$k python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
  python tools/tc_trace.py > gpurun_out/tc_trace_bwd_k$k.txt 2>&1
  cp gpurun_out/tc_trace.bin gpurun_out/tc_trace_bwd_k$k.bin
done
