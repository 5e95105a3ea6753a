#!/bin/bash
cd "$(dirname "$0")/.."
./tools/lutbuild.bin
timeout 300 python -m pytest tests -m gpu -x -q -k "misaligned or tma or kernel_choice" 2>&1 | tail -2
