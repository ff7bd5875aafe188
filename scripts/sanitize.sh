#!/bin/bash
# compute-sanitizer over a representative subset of the GPU tests (run under
# gpurun). memcheck: out-of-bounds / misaligned accesses in the fused level
# kernels (halo lanes, periodic wrap, scalar path, strips, tail), the generic
# executor and the host pipeline; racecheck/synccheck: the kernels use no
# shared memory or CTA barriers except the cooperative tail's grid sync.
set -u
mkdir -p gpurun_out
SEL='run_planar_matches and (cdf97 or dd137) or forward_level_from_image or inverse_level_to_image or host_pipeline or pitched or fused_tail or symmetric_matches and cdf97 or generic_executor'
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_strips.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
