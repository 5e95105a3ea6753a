#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_fused_gather.py -x -q 2>&1 | tail -20
