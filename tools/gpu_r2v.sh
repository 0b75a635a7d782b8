# phase store for split-K blocks (2 x int16 per cell instead of the fp32 W): parity at c2-c5 + timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in c4 c2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['path_roofline']['rest_ms_measured'], d['config']['micro_batch'], {k:(round(v['ms_per_step'],1), round(v['frac'],3)) for k,v in d['roofline']['joint_kernels'].items()})"
done > gpurun_out/v_ab.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -rf --durations=15 2>&1 | tail -25 > gpurun_out/v_tests.txt
