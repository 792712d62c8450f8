# one gpurun call: GPU tests, plain bench, then (ONLY if the plain bench exited 0) the ncu launch list
# and ncu --set full on the top kernels
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --phases > gpurun_out/bench_plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --phases > gpurun_out/ncu_launch.log 2>&1
  echo "ncu1 exit $?" >> gpurun_out/ncu_launch.log
  timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_project|k_render|k_tile_sort|k_adam}" -s ${NCU_S:-40} -c ${NCU_C:-8} -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
else
  echo "plain bench failed: ncu skipped" >> gpurun_out/bench_plain.log
fi
