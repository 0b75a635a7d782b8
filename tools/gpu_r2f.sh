for c in c2 c4; do for m in 0 1; do
  JTFS_BWD_MODE=$m python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c bwdmode=$m', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done; done > gpurun_out/bench_r2f.txt 2>&1
JTFS_BWD_MODE=1 python -m pytest tests -m gpu -q -rf -k "c2-all-music or loss_grad_parity" >> gpurun_out/bench_r2f.txt 2>&1
