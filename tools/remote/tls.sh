python tools/timeline_split.py 4096 4096 0
python tools/timeline_split.py 4096 4096 1 4096
python tools/timeline_split.py 4096 4096 1 1800
python tools/timeline_split.py 8192 8192 0
