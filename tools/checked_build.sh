#!/bin/bash
# The compute-sanitizer stand-in (compute-sanitizer is closed on this GPU pool:
# profiles/r02_compute_sanitizer_refused.txt). Builds paper_1605_02164_b200/libbfvec_checked.so with
# -DBFVEC_CHECKED:
#   * every mbarrier wait has a watchdog (a phase that never completes traps with the barrier
#     address instead of hanging the GPU) -- the synccheck / deadlock part;
#   * the v6 kernel tags every TMEM ring row, (c, s) ring row and G buffer with the row / sub-step
#     it holds, and the consumers verify, before and after reading, that each slot still holds
#     the row they expect -- a premature overwrite (a ring-protocol race) traps -- the racecheck part;
#   * BF_CHECK bounds on the ring slots -- the memcheck part, with the guard-band tests
#     (tests/gpu/test_guards.py) catching out-of-bounds stores to every output;
# then runs the whole GPU suite against it:
#   BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so python -m pytest tests -m gpu -q
set -e
cd "$(dirname "$0")/.."
BFVEC_BUILD_TAG=checked BFVEC_NVCC_EXTRA="-DBFVEC_CHECKED" python paper_1605_02164_b200/build.py
if [ "${1:-}" = "--run" ]; then
  BFVEC_LIB=$PWD/paper_1605_02164_b200/libbfvec_checked.so python -m pytest tests -m gpu -q
fi
