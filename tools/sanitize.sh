#!/bin/bash
# compute-sanitizer over every hot-path kernel (tools/sanitize_run.py) -> gpurun_out/san_<tool>[_<section>].txt,
# and a per-(kernel, source line) hazard digest of each report (san_digest.txt).
mkdir -p gpurun_out
TAG=${TAG:-r02}
python tools/sanitize_run.py > gpurun_out/san_plain_$TAG.txt 2>&1; tail -1 gpurun_out/san_plain_$TAG.txt
run() {  # tool, section(s), lms, timeout, extra
  local out=gpurun_out/san_${1}_${2//,/+}_$TAG.txt
  SAN_ONLY=$2 SAN_LMS=$3 timeout $4 compute-sanitizer --tool $1 $5 --print-limit 400 --target-processes all \
      python tools/sanitize_run.py > $out 2>&1
  echo "$1 [$2] rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run:' $out | tr '\n' ' ')"
}
[ -z "$SKIP_MEM" ] && run memcheck "" "" 1800 "--leak-check no"
for sec in adv fused decode loop topk,rows tiled; do
  run racecheck $sec tri64,six1024 1200 "--racecheck-report all"
done
run synccheck "" "" 1800 ""
run initcheck adv,fused,decode tri64 1500 ""
for f in gpurun_out/san_*_$TAG.txt; do
  echo "== $f"
  grep -E "Error:|Warning:|Barrier error|Uninitialized|Invalid" $f | sed -E 's/0x[0-9a-f]+//g; s/\(ngpulm::DevModel[^)]*\)//g; s/in block \([0-9,]+\)//g' \
      | sort | uniq -c | sort -rn | head -12
done > gpurun_out/san_digest_$TAG.txt
cat gpurun_out/san_digest_$TAG.txt | cut -c1-300
