#!/bin/bash
# compute-sanitizer passes over small frames (run under gpurun): memcheck on a few parity tests,
# racecheck + synccheck on the smoke frame.  Logs land in gpurun_out/sanitize_*.log.
export FGS_SANITIZE=1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/sanitize_memcheck.log \
  python -m pytest tests/test_gpu_parity.py tests/test_scene_io.py -x -q -m gpu \
  -k "golden_pipeline_render or binning_known_answers or row_weights or empty_scene or forced_regrow or device_ingest or row_bands or sparse_scene or dense_tile_with or equal_depth or reference_package" \
  > gpurun_out/sanitize_memcheck.out 2>&1; echo "memcheck rc=$?"
tail -3 gpurun_out/sanitize_memcheck.out; tail -4 gpurun_out/sanitize_memcheck.log
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --log-file gpurun_out/sanitize_$tool.log \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.out 2>&1; echo "$tool rc=$?"
  tail -1 gpurun_out/sanitize_$tool.out; tail -3 gpurun_out/sanitize_$tool.log
done
# racecheck over the sort's dense / tie paths (medium class splitting a > 8192-pair tile, give-up to the tail kernel)
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file gpurun_out/sanitize_racecheck_dense.log \
  python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dense_tile_with or equal_depth_ties_order_by_index and 3000" \
  > gpurun_out/sanitize_racecheck_dense.out 2>&1; echo "racecheck(dense) rc=$?"
tail -1 gpurun_out/sanitize_racecheck_dense.out; tail -3 gpurun_out/sanitize_racecheck_dense.log
# lazy_sort: memcheck + racecheck over the front kernel, the redo sort and the second blend pass
# (mixed scene: half of the fronts are redone; late cluster: fronts cut before a depth cluster)
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/sanitize_memcheck_lazy.log \
  python -m pytest tests/test_lazy_sort.py -x -q -m gpu -k "mixed or late or extras or repeated" \
  > gpurun_out/sanitize_memcheck_lazy.out 2>&1; echo "memcheck(lazy) rc=$?"
tail -1 gpurun_out/sanitize_memcheck_lazy.out; tail -2 gpurun_out/sanitize_memcheck_lazy.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file gpurun_out/sanitize_racecheck_lazy.log \
  python -m pytest tests/test_lazy_sort.py -x -q -m gpu -k "mixed or extras" \
  > gpurun_out/sanitize_racecheck_lazy.out 2>&1; echo "racecheck(lazy) rc=$?"
tail -1 gpurun_out/sanitize_racecheck_lazy.out; tail -2 gpurun_out/sanitize_racecheck_lazy.log
