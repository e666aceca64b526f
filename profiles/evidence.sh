# Round-end evidence run on one B200 (gpurun): GPU tests, smoke, bench lines (C1 headline, C2, C4),
# the reference arm, the ncu launch list and full captures of one training step.
mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c2 --steps 1000 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c4 --steps 100 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c1.json 2> gpurun_out/ref_c1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --profile-steps 2 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -c 7 -o gpurun_out/step_c1 python tests/prof_step.py --warmup 3 --steps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -c 9 -o gpurun_out/step_c2 python tests/prof_step.py --warmup 3 --steps 1 --config c2 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2
