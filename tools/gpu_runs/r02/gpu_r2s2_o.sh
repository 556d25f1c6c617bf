# run O: compute-sanitizer over the round-2 kernel paths
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/o_sanitize.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_r02.py >> gpurun_out/o_sanitize.txt 2>&1
done
