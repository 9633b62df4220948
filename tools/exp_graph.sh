python tools/exp_graph.py 2>&1 | grep "rc="
KRUL_GRAPHS=0 python tools/exp_graph.py 2>&1 | grep "rc="
