timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-policies > gpurun_out/bench_dexp.json 2> gpurun_out/bench_dexp.err
python tools/bench_brief.py gpurun_out/bench_dexp.json | grep -v "None None None"
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_ec_decode_expand -s 10 -c 1 -o gpurun_out/prof_dexp2 -f python tools/profile_step.py > /dev/null 2>&1
python tools/ncu_summary.py --rep gpurun_out/prof_dexp2.ncu-rep | head -14
