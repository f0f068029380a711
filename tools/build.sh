#!/bin/bash
# rebuild the native library from anywhere
cd "$(dirname "$0")/.." && python -c "from paper_2308_06085_b200 import build_native as b; b.build(verbose=False)" 2>&1 | grep -E "rror|warning" -A3 | head -20
