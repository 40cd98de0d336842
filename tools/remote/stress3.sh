for na in 9 8 7 6 5; do echo "na=$na"; TIDE_K1_NA=$na TIDE_K1_PAIRSLOT=0 timeout 60 python tools/stress_detail.py 160000 2048 150 | tail -3; done
