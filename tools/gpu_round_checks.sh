set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_geom.json 2> gpurun_out/bench_geom.err; echo bench=$?
timeout 1200 python tools/microbench_c5.py --device-factor --max-nodes 20000000 --out gpurun_out/c5_default.json > gpurun_out/c5_default.log 2>&1; echo c5=$?
SCENOPT_SWEEP_PRODUCERS=6 timeout 900 python tools/layout_fuzz.py > gpurun_out/fuzz_p6.txt 2>&1; echo fuzz=$?; tail -3 gpurun_out/fuzz_p6.txt
python bench.py --steps 5 --warmup 3 --no-solve --no-cpu-baseline > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep_full python bench.py --steps 5 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1; echo ncull=$?
