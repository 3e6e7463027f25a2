# Round-2 launch lists of configs 0 / 2 / 3 / 4 (ncu per-launch durations: cold caches, serialised).
M="--metrics gpu__time_duration.sum --clock-control none --csv"
ncu $M -c 400 --log-file gpurun_out/l_cfg0.csv python tools/cfg0_once.py 10 > gpurun_out/l0.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg3.csv python tools/cfg0_once.py 10 cfg3 > gpurun_out/l3.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg2.csv python tools/implicit_once.py 20 > gpurun_out/l2.log 2>&1
ncu $M -c 600 --log-file gpurun_out/l_cfg4.csv python tools/ht_timing.py 64 > gpurun_out/l4.log 2>&1
for c in 0 2 3 4; do python tools/ncu_launches.py gpurun_out/l_cfg$c.csv > gpurun_out/r02_cfg${c}_launches.txt; done
