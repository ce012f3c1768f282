# compute-sanitizer over every kernel family (tools/sanitize_case.py); logs in $1
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for case in C1 C4s C4chol C4amg C5 exact; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_case.py $case \
      > "$out/${case}_${tool}.log" 2>&1
    echo "$case $tool exit=$?" | tee -a "$out/summary.txt"
  done
done
