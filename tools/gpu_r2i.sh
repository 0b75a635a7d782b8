python -m pytest tests -m gpu -q -rf -k "c2-all-music or forward_parity or loss_grad_parity or split_k" > gpurun_out/pytest_gpu_r2i.txt 2>&1
for c in c2 c4; do
  python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done > gpurun_out/bench_r2i.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_rowB -c 3 -o gpurun_out/r2i_rowB python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_colA -c 2 -o gpurun_out/r2i_colA python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
