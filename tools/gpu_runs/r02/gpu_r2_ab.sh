# A/B of the headline step: round-1 binding + bench vs current, same box, alternating
cp paper_2601_18150_b200/libfp8q.so ab_old/paper_2601_18150_b200/
for i in 1 2; do
  (cd ab_old && python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > ../gpurun_out/ab_old_$i.json 2>&1)
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ab_new_$i.json 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2_gputests.txt
