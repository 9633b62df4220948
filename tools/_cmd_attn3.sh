python tools/attn_timeline.py 128 8192 0 | sed -n '/MMA \[/,$p' | head -50
