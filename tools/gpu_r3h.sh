# two epilogue groups on alternate tiles (backward, nab = 2 recompute blocks): parity, then A/B (JTFS_TC_EXPT=32 = off)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3h_pytest.txt
run() { timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$1', '$2', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in j.items()})"; }
for c in c2 c4; do run $c twogroup; JTFS_TC_EXPT=32 run $c onegroup; done > gpurun_out/r3h.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_routes.py -m gpu -q -x -k "not c5" 2>&1 | tail -3 >> gpurun_out/r3h_pytest.txt
