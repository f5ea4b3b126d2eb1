for c in C3 C4; do
timeout 900 python bench.py --all-legs --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/alllegs_$c.json 2>gpurun_out/alllegs_$c.err; echo rc=$?; wc -l < gpurun_out/alllegs_$c.json
python -c "import json; d=json.load(open('gpurun_out/alllegs_$c.json')); g=d['gather']; print('$c', d['ms_per_step'], g['headline'], g['fused_check'], g['nccl_check'], json.dumps(g.get('balance')))"
done
