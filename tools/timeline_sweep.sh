#!/bin/bash
# per-CTA timeline of the route kernel under debug variants (see tools/timeline.py)
for f in 0 5; do echo "== TIDE_DEBUG_FLAGS=$f"; TIDE_DEBUG_FLAGS=$f python tools/timeline.py | head -20; done
