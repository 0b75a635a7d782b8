#!/bin/bash
# One GPU call: build, gpu tests, bench, ncu launch list, ncu full capture of the joint kernels.
# usage (on the box, via gpurun): bash tools/gpu_session.sh TAG [CONFIG] [what]
TAG=${1:-r01}; CFG=${2:-c2}; WHAT=${3:-all}; KERNELS=${4:-"k_joint_bwd_tc k_joint_fwd_tc k_joint_bwd_fft"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/${TAG}_build.log; exit 1; }
if [[ $WHAT == *tests* || $WHAT == all ]]; then
  timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
fi
if [[ $WHAT == *bench* || $WHAT == all ]]; then
  timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_${CFG}.json 2> gpurun_out/${TAG}_bench_${CFG}.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench_${CFG}.json | head -c 3000
fi
if [[ $WHAT == *launches* || $WHAT == all ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches_${CFG}.csv \
     python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
if [[ $WHAT == *traffic* ]]; then
  timeout 1500 ncu --set full --clock-control none -k regex:"k_joint|k_gy_reduce" -s 120 -c 34 -o gpurun_out/${TAG}_traffic_${CFG} \
     python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
  # summarise on the box (the report itself is too large to bring back): one step = 1 forward + 1 backward
  python tools/ncu_traffic.py gpurun_out/${TAG}_traffic_${CFG}.ncu-rep $CFG 1 1 gpurun_out/${TAG}_traffic_${CFG}.json > gpurun_out/${TAG}_traffic.log 2>&1
  mkdir -p /tmp/ncu_keep && mv gpurun_out/${TAG}_traffic_${CFG}.ncu-rep /tmp/ncu_keep/
fi
if [[ $WHAT == *full* || $WHAT == all ]]; then
  for K in $KERNELS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s 2 -c 1 -o gpurun_out/${TAG}_${K}_${CFG} \
     python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full_${K}.log 2>&1; echo "ncu full $K rc=$?"
    python tools/ncu_summary.py full gpurun_out/${TAG}_${K}_${CFG}.ncu-rep gpurun_out/${TAG}_${K}_${CFG}_full.txt
    python tools/ncu_lines.py gpurun_out/${TAG}_${K}_${CFG}.ncu-rep 40 > gpurun_out/${TAG}_${K}_${CFG}_lines.txt
    mkdir -p /tmp/ncu_keep && mv gpurun_out/${TAG}_${K}_${CFG}.ncu-rep /tmp/ncu_keep/
  done
fi
