python tools/als_cl_scan.py 64 588 12 10 0:0 1:36 1:24 4:16 4:12 > gpurun_out/ei.txt 2>&1
python tools/als_cl_scan.py 128 300 16 10 0:0 1:49 1:32 4:16 >> gpurun_out/ei.txt 2>&1
python tools/als_cl_scan.py 96 200 8 10 0:0 1:16 4:16 >> gpurun_out/ei.txt 2>&1
python -m pytest tests/test_gpu_cp.py -q -x >> gpurun_out/ei.txt 2>&1
