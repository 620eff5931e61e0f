PEARL_DRAFT_SMS=40 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/dp_40.csv python tools/draft_block_once.py 2 > gpurun_out/dp.log 2>&1
PEARL_DRAFT_SMS=40 timeout 300 python tools/draft_partition_time.py >> gpurun_out/dp.log 2>&1
