# Round-end evidence refresh: GPU suite, smoke, bench (with the CPU baseline), reference arm,
# launch lists of configs 0/2/3/4.
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
M="--metrics gpu__time_duration.sum --clock-control none --csv"
ncu $M -c 400 --log-file gpurun_out/l_cfg0.csv python tools/cfg0_once.py 10 > gpurun_out/l0.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg3.csv python tools/cfg0_once.py 10 cfg3 > gpurun_out/l3.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg2.csv python tools/implicit_once.py 20 > gpurun_out/l2.log 2>&1
ncu $M -c 600 --log-file gpurun_out/l_cfg4.csv python tools/ht_timing.py 64 > gpurun_out/l4.log 2>&1
