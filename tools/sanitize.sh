#!/bin/bash
# compute-sanitizer passes over a parity subset that runs every kernel of a
# training step (run under gpurun, 1 GPU):   bash tools/sanitize.sh
sel="seeded_vs_oracle and 50000 or degenerate or bin_tiles_api or fused_loss or morton or half or densify"
compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$sel" 2>&1 | tail -2
compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "seeded_vs_oracle and 50000 or degenerate" 2>&1 | tail -2
compute-sanitizer --tool synccheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "seeded_vs_oracle and 50000 or degenerate" 2>&1 | tail -2
