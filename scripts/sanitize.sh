#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck over the small-instance GPU parity
# subset (gr17 / eil51): K1 (compact + narrow tables), both K3 kernels, K5,
# K6 and vrp_alns_iterate.  Summaries land in gpurun_out/sanitize_*.log.
#   gpurun --timeout 2400 -- bash scripts/sanitize.sh
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL=(
  "tests/test_gpu_parity.py::test_makespan_family_vs_golden"
  "tests/test_gpu_parity.py::test_decode_vs_golden"
  "tests/test_gpu_parity.py::test_decode_warp_per_chromosome_kernel"
  "tests/test_gpu_parity.py::test_narrow_ready_overflow_falls_back_exactly"
  "tests/test_gpu_repair.py::test_repair_matches_reference_goldens"
  "tests/test_gpu_alns_device.py::test_destroy_kernel_matches_reference_goldens"
  "tests/test_gpu_alns_device.py::test_device_run_alns_matches_reference"
)
K=${SANITIZE_K:-"gr17 or eil51 or toy or reference or overflow"}
for tool in memcheck racecheck; do
  echo "== $tool" | tee gpurun_out/sanitize_$tool.log
  timeout ${SANITIZE_TIMEOUT:-1500} $CS --tool $tool --print-limit 20 --error-exitcode 99 \
    python -m pytest -x -q -p no:cacheprovider -m gpu "${SEL[@]}" -k "$K" \
    >> gpurun_out/sanitize_$tool.log 2>&1
  echo "exit=$?" | tee -a gpurun_out/sanitize_$tool.log
  tail -5 gpurun_out/sanitize_$tool.log
done
