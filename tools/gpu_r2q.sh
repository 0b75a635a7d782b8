# T-layout layer-2 spectra (gather writes T-layout, FromT IFFT; ToT FFT of g_Y2, staged adjoint gather)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -rf -k "not c5 and not c4 and not c3" 2>&1 | tail -5 > gpurun_out/q_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-forward > gpurun_out/q_c4.json 2> gpurun_out/q_c4.err
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-forward > gpurun_out/q_c2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > gpurun_out/q_c4_ncu.log 2>&1
