#!/bin/bash
# compute-sanitizer over a representative subset of the GPU tests (run under
# gpurun). memcheck: out-of-bounds / misaligned accesses in the fused level
# kernels (halo lanes, periodic wrap, scalar path, strips, TMA-staged rows,
# the fused level pair, the wavefront), the generic executor and the host
# pipeline; racecheck/synccheck: the staged kernels' per-warp shared-memory
# rings (mbarrier-signalled bulk copies) and the generic kernel's crops.
set -u
mkdir -p gpurun_out
SEL='run_planar_matches and (cdf97 or dd137) or forward_level_from_image or inverse_level_to_image or host_pipeline or pitched or wavefront or symmetric_fused or generic_executor or tma_staged or level_pair or strip_driver'
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_strips.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
