# B2 ring depth of the backward (JTFS_BWD_NS2 = tiles of lookahead)
run() { python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$1', '$2', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in j.items()})"; }
for c in c4; do
  for e in 3 2 4 5; do JTFS_BWD_NS2=$e run $c ns2=$e; done
done > gpurun_out/r3b.txt 2>&1
JTFS_BWD_NS2=5 JTFS_PLAN_DUMP=1 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-forward 2>&1 | grep "tc block" > gpurun_out/r3b_plan.txt
