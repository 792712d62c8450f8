# Round-2 measurement pass (one gpurun call): GPU suite, the bench lines (C3 default with the CPU
# oracle leg, C2, C4, C5 at N = 1), the reference arm, the ncu launch list of the C3 step and one
# `ncu --set full` capture of the dominant kernels.  Outputs in gpurun_out/r2m_*.
set -u
python -m pytest tests -m gpu -q > gpurun_out/r2m_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/r2m_tests.log)"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print(\"smoke ok\")" > gpurun_out/r2m_smoke.log 2>&1; echo "smoke: $(tail -1 gpurun_out/r2m_smoke.log)"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2m_c3.log 2>&1; echo "c3 rc=$?"
for c in C2 C4 C5; do
  python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2m_$c.log 2>&1; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2m_ref.log 2>&1; echo "ref rc=$?"
if timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m_launches.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-window > gpurun_out/r2m_ncu_launch.log 2>&1; then
  timeout 1200 ncu -f --set full --clock-control none --import-source on \
     -k regex:"k_render_fwd|k_render_bwd|k_project_bwd|k_project|k_tile_sort|k_emit" -s 40 -c 12 \
     -o gpurun_out/r2m_prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-window > gpurun_out/r2m_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
# the realistic window iteration (after insertions: every tile kept), kernel list of 3 iterations
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/r2m_window_launches.csv python scripts/diag_window_iter.py > gpurun_out/r2m_window.log 2>&1
echo "window rc=$?"
# C4 capture of the dominant kernels (for profiles/traffic.json and r2_ncu_summary_c4.txt)
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_render_fwd|k_project|k_tile_sort|k_emit" \
   -s 12 -c 6 -o gpurun_out/r2m_prof_c4 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline \
   > gpurun_out/r2m_ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
