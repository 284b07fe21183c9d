export PYTHONPATH=$PWD
python scripts/walk_time.py 3 5
for V in scr5 scr6 scr7; do BVC_LIB=paper_2302_11825_b200/_build/variants/$V/libbvc_b200.so python scripts/walk_time.py 3 5; done
python scripts/walk_time.py 1 7
for V in dir5 dir7 dir8; do BVC_LIB=paper_2302_11825_b200/_build/variants/$V/libbvc_b200.so python scripts/walk_time.py 1 7; done
