for v in 100000 130 100; do
for c in c2 c4; do
  JTFS_KS1_MIN=$v python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c ks1=$v', round(d['ms_per_step'],2), 'mb', d['config']['micro_batch'], {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done; done > gpurun_out/bench_r2o.txt 2>&1
JTFS_KS1_MIN=130 timeout 900 python -m pytest tests -m gpu -q -rf -k "c2-all-music or split_k" >> gpurun_out/bench_r2o.txt 2>&1
