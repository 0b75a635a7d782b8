# rowT last pass stored straight to global; c1 launch list; full captures of the row/column passes
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -rf -k "c2-all-music or loss_grad_parity or forward_parity or stage" 2>&1 | tail -3 > gpurun_out/s_tests.txt
for c in c4 c2 c4 c2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['path_roofline']['rest_ms_measured'])"
done > gpurun_out/s_ab.txt 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --graph > gpurun_out/s_c1.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s_c1_launches.csv python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv --log-file gpurun_out/s_c2_fft.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_rowT -s 20 -c 1 -o gpurun_out/s_rowT python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_colA -s 12 -c 1 -o gpurun_out/s_colA python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adj_gather_u1 -s 1 -c 1 -o gpurun_out/s_adjg python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
