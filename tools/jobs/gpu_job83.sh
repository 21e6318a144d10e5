#!/bin/bash
# racecheck over the parity tests job 82 did not reach (hybrid, powerlaw, ledger, determinism, ...)
export PYTHONPATH=$PWD
timeout 1700 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_train_gcn_three_stages_wide_features \
  tests/test_gpu_parity.py::test_pipeline_ledger_closed_form \
  tests/test_gpu_parity.py::test_stale_equals_exact_on_chunk_disconnected_graph[id] \
  tests/test_gpu_parity.py::test_stale_equals_exact_on_chunk_disconnected_graph[degree] \
  tests/test_gpu_parity.py::test_deterministic_reruns \
  tests/test_gpu_parity.py::test_live_reference_gcnii_three_stages \
  tests/test_gpu_parity.py::test_invalid_arguments_raise \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_gcn_hyb_s2g2] \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_gcnii_hyb_s2g2] \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_gcnii_hyb_s1g3_sync] \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_gcn_hyb_s3g2_hist] \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_sage_hyb_s2g2] \
  tests/test_gpu_parity.py::test_train_hybrid_matches_reference[train_sage_hyb_s1g2_hist] \
  tests/test_gpu_parity.py::test_train_gcn_pipeline_powerlaw_graph \
  tests/test_gpu_parity.py::test_train_hybrid_powerlaw_graph -q -m gpu -p no:cacheprovider > gpurun_out/j83_racecheck.txt 2>&1; echo "racecheck rc=$?"; grep -E "passed|failed|SUMMARY|skipped" gpurun_out/j83_racecheck.txt | tail -3
