#!/bin/bash
for f in 0 2 32; do echo "== TIDE_DEBUG_FLAGS=$f"; TIDE_DEBUG_FLAGS=$f python tools/timeline.py | grep -E "stream_done|epi_done|end |MMA"; done
