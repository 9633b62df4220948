timeout 600 python -m pytest tests -m gpu -x -q -k "attn or attention or fa or prefill or restore or turn or batch" 2>&1 | tail -2
for v in 1 2; do echo "== KRUL_ATTN_V=$v"; KRUL_ATTN_V=$v python tools/attn_bench.py 2>&1 | grep -E "target=(0|8):"; done
python tools/attn_timeline.py 128 8192 0 | sed -n '/softmaxA/,$p' | head -24
