timeout 900 python tools/paper_style.py 20 > gpurun_out/paper_style.jsonl 2>&1
