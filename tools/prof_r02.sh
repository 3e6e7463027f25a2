# Round-2 evidence for the bench dominant kernel (config 1, als_w): plain bench line,
# the launch list of the same bench command, one full ncu capture of the ALS kernel.
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
TP_ALS_NONCOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/r02_launches.log 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches.txt
TP_ALS_NONCOOP=1 ncu --set full --clock-control none --import-source on -k regex:als_ -c 1 -o gpurun_out/r02_als_full \
  python tools/als_once.py > gpurun_out/r02_als_full.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
