ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv scripts/dbg/gran3_bench > gpurun_out/gran3.csv 2>&1
grep -E "dram__|gpu__time" gpurun_out/gran3.csv | awk -F'","' '{print $5, $(NF-2), $NF}'
bash scripts/gpu_ab.sh 4
