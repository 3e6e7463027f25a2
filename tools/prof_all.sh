set -x
M="--metrics gpu__time_duration.sum --clock-control none --csv"
ncu $M -c 400 --log-file gpurun_out/l_cfg0.csv python tools/cfg0_once.py 10 > gpurun_out/l0.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg3.csv python tools/cfg0_once.py 10 cfg3 > gpurun_out/l3.log 2>&1
ncu $M -c 400 --log-file gpurun_out/l_cfg2.csv python tools/implicit_once.py 20 > gpurun_out/l2.log 2>&1
ncu $M -c 600 --log-file gpurun_out/l_cfg4.csv python tools/ht_timing.py 64 > gpurun_out/l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:als_tiny8 --launch-skip 3 -c 1 -o gpurun_out/tiny8 python tools/cfg0_once.py 6 > gpurun_out/t8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:circ_gs --launch-skip 1 -c 1 -o gpurun_out/circgs python tools/implicit_once.py 20 > gpurun_out/cg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jacobi_eigh --launch-skip 5 -c 1 -o gpurun_out/jac0 python tools/ht_timing.py 64 > gpurun_out/j0.log 2>&1
