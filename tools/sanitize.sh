#!/bin/bash
# compute-sanitizer passes over small end-to-end cases (GPU box): memcheck,
# racecheck (shared-memory hazards), synccheck, initcheck.
set -u
PY='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -c "$PY" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -m1 'ERROR SUMMARY' gpurun_out/san_$tool.log)"
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "load_tokens or partition_gpu_matches_host or checkpoint or large_k or conservation or resident or set_phi or tree_api or pinned or heavy_word or document_groups" > gpurun_out/san_memcheck_tests.log 2>&1
echo "memcheck(tests) rc=$? $(grep -m1 'ERROR SUMMARY' gpurun_out/san_memcheck_tests.log) $(tail -1 gpurun_out/san_memcheck_tests.log)"
# K2 heavy-word pieces + K3 document groups on corpora with heavy words
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 99 python tools/probes/k23_heavy_groups.py > gpurun_out/san_memcheck_k23.log 2>&1
echo "memcheck(k2/k3) rc=$? $(grep -m1 'ERROR SUMMARY' gpurun_out/san_memcheck_k23.log)"
# phases: word and document-block phases, the overlapped sample export, doc-major transfers
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_phases.py tests/test_gpu_block_phases.py -m gpu -x -q > gpurun_out/san_memcheck_phases.log 2>&1
echo "memcheck(phases) rc=$? $(grep -m1 'ERROR SUMMARY' gpurun_out/san_memcheck_phases.log) $(tail -1 gpurun_out/san_memcheck_phases.log)"
