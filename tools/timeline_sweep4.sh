#!/bin/bash
for pf in 0 2 4 8 12; do echo "== prefetch $pf"; TIDE_PREFETCH=$pf python tools/timeline.py | grep -E "stream|epi_done|end |MMA"; done
