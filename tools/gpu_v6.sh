# round-2 v6 measurement set at HEAD: GPU suite, smoke, default (c4) and c2 bench lines, c4 launch list with DRAM bytes,
# c4 tensor-pipe counters of the joint launches
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/y_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=5 > gpurun_out/y_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/y_c4_bench.json 2> gpurun_out/y_c4_bench.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/y_c2_bench.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/y_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_joint --csv --log-file gpurun_out/y_c4_tensor.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
