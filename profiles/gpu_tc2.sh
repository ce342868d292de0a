mkdir -p gpurun_out
export KVMIX_TC_DEBUG=1
timeout 600 python -m pytest tests/test_attention_tc_gpu.py -q 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20 > gpurun_out/tc_tests.log
KVMIX_TC=1 timeout 300 python profiles/attend_time.py > gpurun_out/attend_time.log 2>&1
KVMIX_TC=1 SHAPE=8,8,4,32768 timeout 300 python profiles/attend_time.py > gpurun_out/attend_time_gqa.log 2>&1
KVMIX_TC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python profiles/drive_attend.py > gpurun_out/drive.log 2>&1
KVMIX_TC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_tc -s 1 -c 1 -o gpurun_out/tc_prof2 python profiles/drive_attend.py 0 > gpurun_out/drive2.log 2>&1
