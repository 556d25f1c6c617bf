# run P: racecheck with every report printed (unique locations summarised locally)
timeout 900 compute-sanitizer --tool racecheck --print-limit 1000 python tools/sanitize_r02.py > gpurun_out/p_race.txt 2>&1
