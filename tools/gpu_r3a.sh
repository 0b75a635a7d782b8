# issuer-wait experiments (JTFS_TC_EXPT bits 8 spin / 16 single fence; JTFS_TC_FEXPT bits 16 / 32), results unchanged
run() { python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$1', '$2', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in j.items()})"; }
for c in c2 c4; do
  for e in 0 8 16 24; do JTFS_TC_EXPT=$e run $c bexpt=$e; done
  for e in 16 32 48; do JTFS_TC_FEXPT=$e run $c fexpt=$e; done
done > gpurun_out/r3a.txt 2>&1
JTFS_TC_EXPT=24 JTFS_TC_FEXPT=48 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r3a_pytest.txt
