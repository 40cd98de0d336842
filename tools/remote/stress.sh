export TIDE_K1_PAIRSLOT=0
echo "base";   timeout 120 python tools/stress_k1.py 800 160000x1024 2>&1 | grep reps
echo "pdl0";   TIDE_PDL=0 timeout 120 python tools/stress_k1.py 800 160000x1024 2>&1 | grep reps
echo "nw3";    TIDE_NW=3 timeout 120 python tools/stress_k1.py 800 160000x1024 2>&1 | grep reps
echo "nw2";    TIDE_NW=2 timeout 120 python tools/stress_k1.py 800 160000x1024 2>&1 | grep reps
echo "d2048";  timeout 120 python tools/stress_k1.py 800 160000x2048 2>&1 | grep reps
echo "pair d1024"; TIDE_K1_PAIRSLOT=1 timeout 120 python tools/stress_k1.py 800 160000x1024 2>&1 | grep reps
