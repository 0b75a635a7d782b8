python bench.py > gpurun_out/bench_c4_r2l.json 2> gpurun_out/bench_c4_r2l.err
python bench.py --config c2 > gpurun_out/bench_c2_r2l.json 2> gpurun_out/bench_c2_r2l.err
python bench.py --config c1 --graph --steps 50 > gpurun_out/bench_c1_r2l.json 2> gpurun_out/bench_c1_r2l.err
python bench.py --config c3 --steps 3 --no-e2e --metamer 100 > gpurun_out/bench_c3_r2l.json 2> gpurun_out/bench_c3_r2l.err
python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e --no-forward --metamer 100 --metamer-init colored > gpurun_out/bench_c3col_r2l.json 2> gpurun_out/bench_c3col_r2l.err
python bench.py --config c5 --steps 2 --warmup 3 --no-forward > gpurun_out/bench_c5_r2l.json 2> gpurun_out/bench_c5_r2l.err
python bench.py --impl reference --steps 1 > gpurun_out/bench_ref_c4_r2l.json 2> gpurun_out/bench_ref_c4_r2l.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2l_c4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2l_c2_launches.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_joint --csv --log-file gpurun_out/r2l_c4_tensor.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
