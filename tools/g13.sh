set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k "regex:k_big|k_spmv|k_update|k_pupdate" -c 24 --csv python tools/prof_nb32.py > gpurun_out/g13_nb32_ncu.csv 2> gpurun_out/g13_err.log; echo "rc=$?"
