python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for e in 0 1 2 4 3 7; do
  JTFS_TC_EXPT=$e python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/expt_$e.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/expt_$e.json')); print('expt $e', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['roofline']['joint_kernels'].items()})"
done
