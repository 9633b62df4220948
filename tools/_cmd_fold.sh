for f in 8 1 2 4; do for pre in 3 1; do echo -n "first $f pre $pre: "; KRUL_FOLD_PRE=$pre KRUL_FOLD_FIRST=$f KRUL_FOLD_PITCH=512 FOLD_LOOP=200 python tools/fold_bench.py | tail -1; done; done
KRUL_FOLD_FIRST=2 FOLD_TIMELINE=2 KRUL_FOLD_PITCH=512 python tools/fold_bench.py > /tmp/tl.txt; grep "^cta" /tmp/tl.txt | head -4
timeout 300 python -m pytest tests -m gpu -x -q -k "fold or est" 2>&1 | tail -1
