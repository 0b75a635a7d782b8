timeout 900 python -m pytest tests -m gpu -q -rf -k "stage or forward_parity or loss_grad_parity" > gpurun_out/pytest_gpu_r2n.txt 2>&1
for c in c2 c4; do
  python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --no-forward 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); j=d['roofline']['joint_kernels']
print('$c', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in j.items()})"
done > gpurun_out/bench_r2n.txt 2>&1
python tools/fft_vs_cufft.py c4 4 > gpurun_out/fft_vs_cufft_c4_n.txt 2>&1
