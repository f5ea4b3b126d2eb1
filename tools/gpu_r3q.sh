timeout 900 python bench.py --all-legs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/alllegs.json 2>gpurun_out/alllegs.err; echo rc=$?
cat gpurun_out/alllegs.json | head -c 3000; echo
grep -v '^frame' gpurun_out/alllegs.err | tail -5
