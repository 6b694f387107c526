#!/bin/bash
# compute-sanitizer over the GPU kernels (run on the GPU box): memcheck over the kernel and
# parity suites, racecheck / synccheck over the single-kernel suite (shared-memory races and
# barrier misuse in the tcgen05 / TMA / mbarrier kernels).  Logs -> gpurun_out/sanitize_*.log
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
export ELATTN_PDL=${ELATTN_PDL:-1}
$CS --tool memcheck --leak-check no --report-api-errors no --print-limit 50 \
    python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_mha_gpu.py -q -x \
    -k "not full_size and not (garbage_workspace and (75 or 320))" > "$out/sanitize_memcheck.log" 2>&1
echo "memcheck rc=$?"
$CS --tool racecheck --racecheck-report all --print-limit 50 \
    python -m pytest tests/test_kernels_gpu.py -q -x -k "decode_vs_torch and (64-32-512 or 16-77) or gemm_vs_torch and 128-128 or tf32x3 and 128-128 or splitk and 77-192 or ragged_schedules and 5-64 or fused_query_expansion and (4-1024 or 200-512)" \
    > "$out/sanitize_racecheck.log" 2>&1
echo "racecheck rc=$?"
$CS --tool synccheck --print-limit 50 \
    python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm_vs_torch and 128-128 or tf32x3 and 128-128 or splitk and 77-192 or fused_query_expansion and (4-1024 or 200-512)" \
    > "$out/sanitize_synccheck.log" 2>&1
echo "synccheck rc=$?"
for f in memcheck racecheck synccheck; do echo "== $f"; tail -5 "$out/sanitize_$f.log"; done
