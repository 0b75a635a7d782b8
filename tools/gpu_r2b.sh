# r2b: GPU tests (fast set) after the path-shard refactor, c4 bench (default), c2/c1/c3 lines, ncu launch lists
set -x
python -m pytest tests -m gpu -q -rf -k "not test_large_forward_and_gradient" > gpurun_out/pytest_gpu_r2b.txt 2>&1
python bench.py > gpurun_out/bench_c4_r2b.json 2> gpurun_out/bench_c4_r2b.err
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2_r2b.json 2> gpurun_out/bench_c2_r2b.err
python bench.py --config c1 --graph --steps 50 > gpurun_out/bench_c1_r2b.json 2> gpurun_out/bench_c1_r2b.err
python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e --metamer 100 > gpurun_out/bench_c3_r2b.json 2> gpurun_out/bench_c3_r2b.err
python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e --no-forward --metamer 100 --metamer-init colored > gpurun_out/bench_c3col_r2b.json 2> gpurun_out/bench_c3col_r2b.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2b_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > gpurun_out/r2b_c4_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2b_c2_launches.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > gpurun_out/r2b_c2_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_joint --csv --log-file gpurun_out/r2b_c2_tensor.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > gpurun_out/r2b_c2_tensor.log 2>&1
