#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py; one summary file per tool under gpurun_out/.
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; tail -1 gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  filt="--kernel-name kns=ckv"; [ "$tool" = "initcheck" ] && filt=""  # initcheck must see torch's init writes
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all $filt \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
