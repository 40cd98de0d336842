echo "pair d2048";   timeout 100 python tools/stress_detail.py 160000 2048 200 | tail -4
echo "pair d4096";   timeout 100 python tools/stress_detail.py 160000 4096 100 | tail -4
echo "nopair d4096"; TIDE_K1_PAIRSLOT=0 timeout 100 python tools/stress_detail.py 160000 4096 100 | tail -4
echo "nopair d2048 nw3"; TIDE_NW=3 TIDE_K1_PAIRSLOT=0 timeout 100 python tools/stress_detail.py 160000 2048 200 | tail -4
echo "nopair d2048 gran16"; TIDE_K1_GRAN=16 TIDE_K1_PAIRSLOT=0 timeout 100 python tools/stress_detail.py 160000 2048 200 | tail -4
