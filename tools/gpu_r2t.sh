# rowT float32 A/B: default 2 rows x 512 threads (SMEM twiddles) vs JTFS_ROWT_ALT (1 row x 256, L1 twiddles, 4 CTAs/SM)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
JTFS_ROWT_ALT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf -k "loss_grad_parity or forward_parity" 2>&1 | tail -2 > gpurun_out/t_tests.txt
for v in def alt def alt; do
  if [ $v = alt ]; then export JTFS_ROWT_ALT=1; else unset JTFS_ROWT_ALT; fi
  for c in c4 c2; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-forward --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['path_roofline']['rest_ms_measured'])"
  done
done > gpurun_out/t_ab.txt 2>&1
JTFS_ROWT_ALT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv --log-file gpurun_out/t_c2_fft_alt.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
