for c in f73873c b273415 3b1e480 04a77a3; do (cd bisect_$c && TAG=$c python scripts/c3_time.py 2>&1 | tail -1); done
TAG=head python scripts/c3_time.py
TAG=head_hostsegs ADAPT_HOST_SEGS=1 python scripts/c3_time.py
