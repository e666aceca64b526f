# Round evidence on one B200 (gpurun): GPU tests, smoke, bench lines (C1 headline + fast
# modes, C2, C3 at global batch 4096, C4, C5), the reference arm, the ncu launch list of the
# C1 bench and full captures of one step (C1, C2, C4), summarised on the box; only the C1
# report is kept so gpurun_out stays under the copy-back limit.
#   gpurun --timeout 3000 -- 'bash profiles/evidence.sh r02c'
mkdir -p gpurun_out
TAG=${1:-r02c}
set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --gemm-planes 2 --no-cpu-baseline > gpurun_out/bench_c1_bf16x2.json 2> gpurun_out/bench_c1_bf16x2.err
python bench.py --gemm-planes 1 --no-cpu-baseline > gpurun_out/bench_c1_bf16.json 2> gpurun_out/bench_c1_bf16.err
python bench.py --config c2 --steps 1000 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 4 --profile-steps 2 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 4 --profile-steps 2 --gemm-planes 2 --no-cpu-baseline > gpurun_out/bench_c3_bf16x2.json 2> gpurun_out/bench_c3_bf16x2.err
python bench.py --config c4 --steps 100 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c5 --steps 100 --e2e-steps 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c1.json 2> gpurun_out/ref_c1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --profile-steps 2 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -c 8 -o gpurun_out/step_c1 python tests/prof_step.py --warmup 3 --steps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -c 9 -o gpurun_out/step_c2 python tests/prof_step.py --warmup 3 --steps 1 --config c2 > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none -c 11 -o gpurun_out/step_c4 python tests/prof_step.py --warmup 3 --steps 1 --config c4 > gpurun_out/ncu_full4.log 2>&1
python profiles/summarize_ncu.py gpurun_out/step_c1.ncu-rep ${TAG} && mv profiles/${TAG}_ncu.json gpurun_out/
python profiles/summarize_ncu.py gpurun_out/step_c2.ncu-rep ${TAG}_c2 && mv profiles/${TAG}_c2_ncu.json gpurun_out/
python profiles/summarize_ncu.py gpurun_out/step_c4.ncu-rep ${TAG}_c4 && mv profiles/${TAG}_c4_ncu.json gpurun_out/
rm -f gpurun_out/step_c2.ncu-rep gpurun_out/step_c4.ncu-rep
# compute-sanitizer (racecheck / synccheck / memcheck over one C1 step), if the pool allows it
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_step.py > gpurun_out/sanitize_$tool.log 2>&1; echo "EXIT $?" >> gpurun_out/sanitize_$tool.log
done
du -sh gpurun_out/*
tail -2 gpurun_out/pytest_gpu.log
tail -1 gpurun_out/smoke.log
