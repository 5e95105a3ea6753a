#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_apot2.py -x -q 2>&1 | tail -15
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
