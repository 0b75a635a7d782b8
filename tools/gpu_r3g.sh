timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3g_pytest.txt
run() { python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$1', '$2', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in j.items()})"; }
for c in c2 c4; do run $c hoist; done > gpurun_out/r3g.txt 2>&1
