# determinism of the 3xTF32 route with the pre-split W and the (3, 4, 3) ring
export STRESS_F32=1
for s in 65536x4096 16384x8192 100000x1024 5000x4096 160000x256; do
  timeout 300 python tools/stress_k1.py 200 $s 2>&1 | tail -1
done
