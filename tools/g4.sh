set -u
mkdir -p gpurun_out
CMD="python bench.py --config c2 --warmup 1 --no-cpu-baseline --profile-only --profile-reps 1"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g4_bench_wt.json 2> gpurun_out/g4_bench_wt.err; echo "bench rc=$?"
$CMD > gpurun_out/g4_plain.log 2>&1; echo "plain rc=$?"
prof() {  # tag env regex
  env $2 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$3" -c 2 -o /tmp/$1 $CMD > gpurun_out/$1_ncu.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ls -la /tmp/$1.ncu-rep
}
prof g4_wt "MPB_WT=1" "k_bjac_wt|k_update_first_wt"
prof g4_old "MPB_WT=0" "k_bjac_tile|k_update_first"
du -sh gpurun_out
