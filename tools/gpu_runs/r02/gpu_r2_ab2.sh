python tools/host_probe.py > gpurun_out/host_probe.txt 2>&1
cp paper_2601_18150_b200/libfp8q.so ab_old/paper_2601_18150_b200/
# new bench, old package
mkdir -p /tmp/nb && cp bench.py /tmp/nb/ && cp -r ab_old/paper_2601_18150_b200 /tmp/nb/ && cp -r synth oracle /tmp/nb/ && cp MEASURED_PEAKS.json /tmp/nb/ 2>/dev/null
sed -i 's/, strict=False)/)/' /tmp/nb/bench.py
(cd /tmp/nb && python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > $GRAFT_REPO_ROOT/gpurun_out/ab_newbench_oldpkg.json 2>&1)
(cd ab_old && python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > ../gpurun_out/ab_old_3.json 2>&1)
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ab_new_3.json 2>&1
