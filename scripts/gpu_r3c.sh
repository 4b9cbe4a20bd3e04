python scripts/exp_overlap.py 5 262144 65536,32768,16384
python scripts/exp_overlap.py 5 1048576 131072,65536
python scripts/exp_overlap.py 3 262144 65536,32768
python scripts/exp_overlap.py 1 262144 65536,32768
