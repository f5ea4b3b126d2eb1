# Round evidence on one B200: parity tests, smoke, bench lines (C3 + every config), ncu launch
# list of the bench command and one full capture of rc/pair/bp on C3.
set -x
mkdir -p gpurun_out/configs
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
for c in C0 C2 C4 C5 C5i C6 C6p; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/configs/bench_$c.json 2> gpurun_out/configs/bench_$c.err; echo $c rc=$?
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rc_kernel|bp_kernel|pair_kernel|split_sum" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 300 python tools/prof_bp.py C3 2 > gpurun_out/plain_prof.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bp_kernel|rc_kernel|pair_kernel" -s 3 -c 3 \
    -o gpurun_out/prof_full python tools/prof_bp.py C3 2 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
