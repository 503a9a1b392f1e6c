#!/bin/bash
# quick GPU check: gemm unit tests, parity tests, smoke, short bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -m pytest tests/test_gpu_gemm.py -q 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
