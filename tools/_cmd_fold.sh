python tools/fold_bench.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fold -c 2 -o gpurun_out/prof_fold -f python tools/fold_bench.py > /dev/null 2>&1
python tools/ncu_summary.py --rep gpurun_out/prof_fold.ncu-rep
python tools/ncu_hot.py gpurun_out/prof_fold.ncu-rep 20
