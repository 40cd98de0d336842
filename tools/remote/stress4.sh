export TIDE_K1_PAIRSLOT=0
for d in 2048 1024; do echo "d=$d"; timeout 60 python tools/stress_detail.py 160000 $d 150 | tail -3; done
echo "na=7"; TIDE_K1_NA=7 timeout 60 python tools/stress_detail.py 160000 2048 150 | tail -3
unset TIDE_K1_PAIRSLOT
timeout 300 python tools/stress_k1.py 150 160000x256 160000x2048 100000x1024 65536x4096 2>&1 | grep reps
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks_sustained']['ms_per_launch'])"; done
