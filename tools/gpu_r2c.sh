set -x
python -m pytest tests -m gpu -q -rf -k "not test_large_forward_and_gradient" > gpurun_out/pytest_gpu_r2c.txt 2>&1
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py spec > gpurun_out/sanitize_${t}_spec.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${t}_spec.txt
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py c1 > gpurun_out/sanitize_racecheck_c1.txt 2>&1; echo "exit $?" >> gpurun_out/sanitize_racecheck_c1.txt
