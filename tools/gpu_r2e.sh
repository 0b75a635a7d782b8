for c in c2 c4; do for lanes in 1 2; do for e in 0 3; do
  JTFS_LANES=$lanes JTFS_TC_FEXPT=$e python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c lanes=$lanes fexpt=$e', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done; done; done > gpurun_out/bench_r2e.txt 2>&1
