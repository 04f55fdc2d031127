# normalize export A/B on the B200: detect tests, 8K detect timing with the
# one-compare map (default) and the search form (SOBEL5_NORM_ONE_STEP=0),
# PDL off, and the ncu launch list of one normalize call
python -m pytest tests/test_gpu_detect.py tests/test_gpu_stress.py tests/test_gpu_sobel3.py -x -q > gpurun_out/det_tests.log 2>&1; echo rc=$? >> gpurun_out/det_tests.log
python tools/detect_time.py > gpurun_out/det1.txt 2>&1
SOBEL5_NORM_ONE_STEP=0 python tools/detect_time.py > gpurun_out/det0.txt 2>&1
SOBEL5_PDL=0 python tools/detect_time.py > gpurun_out/det_nopdl.txt 2>&1
python tools/detect_time.py >> gpurun_out/det1.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:norm_map -c 6 --csv --log-file gpurun_out/det_launch2.csv python tools/detect_time.py > /dev/null 2>&1
echo done
