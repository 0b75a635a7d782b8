timeout 1500 python -m pytest tests -m gpu -q -rf -k "stage or forward_parity or loss_grad_parity or c2-all-music or c4-b0-11 or split_k or metamer or cli" > gpurun_out/pytest_gpu_r2m.txt 2>&1
for c in c2 c4; do
  python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done > gpurun_out/bench_r2m.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv --log-file gpurun_out/r2m_c4_fft.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
