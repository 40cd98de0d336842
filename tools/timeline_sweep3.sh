#!/bin/bash
echo "== tc2 scan"; python tools/timeline.py
echo "== tc2 noscan"; TL_NOSCAN=1 python tools/timeline.py
echo "== tc1 scan"; TIDE_K1_SINGLE=1 python tools/timeline.py
echo "== tc1 noscan"; TIDE_K1_SINGLE=1 TL_NOSCAN=1 python tools/timeline.py
