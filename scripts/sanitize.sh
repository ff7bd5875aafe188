#!/bin/bash
# compute-sanitizer over a representative subset of the GPU tests (run under
# gpurun). memcheck: out-of-bounds / misaligned accesses in the fused level
# kernels (halo lanes, periodic wrap, scalar path, strips, TMA-staged rows,
# the fused level pair with packed FP32), the compiled symmetric crop kernel
# (ghost cells, PDL wait-at-end chain), the generic executor in float32 and
# float64, image batches and the host pipeline; racecheck/synccheck: the
# staged kernels' per-warp shared-memory rings (mbarrier-signalled bulk
# copies) and the crop kernels' shared-memory tiles.
set -u
mkdir -p gpurun_out
SEL='run_planar_matches and (cdf97 or dd137) or forward_level_from_image or inverse_level_to_image or host_pipeline or pitched or symmetric or generic_executor or tma_staged or level_pair or strip_driver or float64 or batch_equals'
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_strips.py tests/test_float64.py tests/test_batch.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
