python -m pytest tests -m gpu -q -rf -k "c2-all-music or parity or split_k or c4-b0-11 or repeatability" > gpurun_out/pytest_gpu_r2g.txt 2>&1
for c in c2 c4; do
  python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done > gpurun_out/bench_r2g.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:phiT --csv --log-file gpurun_out/r2g_c4_phiT.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
