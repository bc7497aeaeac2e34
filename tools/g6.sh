set -u
mkdir -p gpurun_out
CMD="python bench.py --config c2 --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
prof() {  # tag env regex count
  env $2 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$3" -c $4 -o /tmp/$1 $CMD > gpurun_out/$1_ncu.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>/dev/null
}
prof g6_last "MPB_WT=0" "k_bjac_tileIfLb0ELb1E" 1
prof g6_upd "MPB_WT=0" "k_update_firstIfLb0E" 1
prof g6_spmv "MPB_WT=0" "k_spmv_pq" 1
du -sh gpurun_out
