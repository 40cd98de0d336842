timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/final3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final3_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final3_smoke.log
timeout 600 python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final3_ref.json 2> gpurun_out/final3_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/final3_tests.log; tail -2 gpurun_out/final3_smoke.log
