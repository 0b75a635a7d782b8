# what bounds the joint kernels per block at c4: ncu launch lists under timing experiments (results invalid
# by design: JTFS_TC_EXPT 1 = no backward epilogue math, 2 = no backward B copies after the first tile,
# 4 = no GEMM2 MMAs; JTFS_TC_FEXPT 4 = no forward B copies after the first tiles, 2 = no W/phase stores)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_joint --csv --log-file gpurun_out/z_$1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-forward > /dev/null 2>&1; }
run base
JTFS_TC_EXPT=2 JTFS_TC_FEXPT=4 run nocopy
JTFS_TC_EXPT=1 run noepi
JTFS_TC_EXPT=4 JTFS_TC_FEXPT=2 run nomma2_nostore
