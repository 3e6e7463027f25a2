# Round-end evidence for the bench's dominant kernel (config 1): plain bench run, the
# launch list of the same bench command, one full ncu capture of the ALS kernel.
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/b_plain.json 2> gpurun_out/b_plain.err
TP_ALS_NONCOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/l_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/l_bench.log 2>&1
TP_ALS_NONCOOP=1 ncu --set full --clock-control none --import-source on -k regex:als_ -c 1 -o gpurun_out/als_full \
  python tools/als_once.py > gpurun_out/als_full.log 2>&1
