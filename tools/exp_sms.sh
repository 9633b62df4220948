for v in 0 24 40 56; do KRUL_NEW_SMS=$v timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-policies > gpurun_out/bench_sms_$v.json 2>/dev/null; python3 -c "
import json; b=json.load(open('gpurun_out/bench_sms_$v.json')); print('new_sms=$v', b['ttft_p50_ms'], b['config']['r_c'], round(b['restore']['compute_ms'],2), round(b['restore']['load_ms'],2), b['roofline']['achieved'])"; done
