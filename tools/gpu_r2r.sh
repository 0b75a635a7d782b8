# row-pass occupancy A/B (JTFS_ROWT_OLD=1: round-2 4 rows x 1024 threads / 2 x 512 with SMEM twiddles)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -rf -k "c2-all-music or loss_grad_parity or forward_parity" 2>&1 | tail -3 > gpurun_out/r_tests.txt
for v in new old new old; do
  if [ $v = old ]; then export JTFS_ROWT_OLD=1; else unset JTFS_ROWT_OLD; fi
  for c in c4 c2; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['path_roofline']['rest_ms_measured'])"
  done
done > gpurun_out/r_ab.txt 2>&1
unset JTFS_ROWT_OLD
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv --log-file gpurun_out/r_c2_fft_new.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
JTFS_ROWT_OLD=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv --log-file gpurun_out/r_c2_fft_old.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
