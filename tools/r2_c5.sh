#!/bin/bash
# C5 exact-phase iteration: GEMM-screen parity tests, full-size C5, probe (staged vs per-warp L2 path)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_tc.py tests/test_gpu_fuzz.py "tests/test_gpu_fullsize.py::test_c5_full_size_tensor_core_screen" > gpurun_out/c5_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/c5_tests.log
timeout 600 python tools/probe_c5.py 2>&1 | tail -5
