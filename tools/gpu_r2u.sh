# float32 row passes 1 row x 256 threads (default now); GPU parity subset; c4/c2 timing; c4 launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_metamer.py -m gpu -x -q -rf -k "not c5 and not c4 and not c3" 2>&1 | tail -2 > gpurun_out/u_tests.txt
for c in c4 c2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['path_roofline']['rest_ms_measured'])"
done > gpurun_out/u_ab.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/u_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
