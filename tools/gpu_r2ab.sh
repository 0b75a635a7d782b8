# gathers without 64-bit divides (shifts; 32-bit in-row indices): parity + timing + per-kernel times
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -rf -k "not c5 and not c4-b0" 2>&1 | tail -4 > gpurun_out/ab_tests.txt
for c in c4 c2 c4 c2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['path_roofline']['rest_ms_measured'],2), d['config']['micro_batch'], {k:(round(v['ms_per_step'],1), round(v['frac'],3)) for k,v in d['roofline']['joint_kernels'].items()})"
done > gpurun_out/ab_ab.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather|phase|modulus|phiT" --csv --log-file gpurun_out/ab_c4_rest.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
