# forward epilogue bound? ncu launch list with JTFS_TC_FEXPT=8 (no modulus / phi_F math; results invalid by design)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
JTFS_TC_FEXPT=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_joint_fwd --csv --log-file gpurun_out/z_noepif.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_joint_fwd --csv --log-file gpurun_out/z_basef.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1
