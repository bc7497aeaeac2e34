mkdir -p gpurun_out
: > gpurun_out/parity_r01n.jsonl
for spec in "c1 uniform" "c1 fixed-low" "c2 fixed-low" "c4 fixed-low" "c4 adaptive-hl:10" "c5 fixed-low --max-iter 12" "c3 adaptive-lh:1e-6"; do
  set -- $spec
  cfg=$1; pol=$2; shift 2
  timeout 1500 python tools/fullsize_parity.py $cfg --policy $pol "$@" >> gpurun_out/parity_r01n.jsonl 2>> gpurun_out/parity_r01n.err
  echo "$cfg $pol rc=$?"
done
