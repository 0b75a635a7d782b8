# backward epilogue with 8 warps x 16 rows (JTFS_BW_EPIW=8) instead of 16 x 8: parity, then timing
JTFS_NVCC_EXTRA=-DJTFS_BW_EPIW=8 python -c "
import sys; sys.path.insert(0,'.')
from paper_2602_11896_b200 import build as b; b.build(force=True)" > gpurun_out/r3f_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3f_pytest.txt
run() { python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$1', '$2', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in j.items()})"; }
for c in c2 c4; do run $c epiw8; done > gpurun_out/r3f.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -q -x -k "c2" 2>&1 | tail -3 >> gpurun_out/r3f_pytest.txt
