#!/bin/bash
# same-box calibration: TMA streaming probe (upper bound) vs the kernel timeline
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv,noheader
./tools/tma_probe 2>&1 | grep -E "mode=0 kq=1 tiles=4 ns= 9 wload=1|mode=2 kq=4 tiles=4 ns= 9 wload=0"
for v in "$@"; do echo "== $v"; env $v python tools/timeline.py | grep -E "stream|epi_done|end |MMA"; done
