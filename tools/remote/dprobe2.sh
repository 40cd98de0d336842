export TIDE_DEBUG_PLAN=1
python tools/decode_exp.py base 2>&1 | tail -3
for c in 256 320 384 448 512; do TIDE_DECODE_COLS=$c python tools/decode_exp.py cols$c 2>&1 | tail -3; done
