python scripts/c3_time.py
TAG=host_segs ADAPT_HOST_SEGS=1 python scripts/c3_time.py
TAG=two ADAPT_TWO_LEVEL=1 python scripts/c3_time.py
TAG=nosmall ADAPT_NO_SMALL=1 python scripts/c3_time.py
ADAPT_TRACE_HOST=1 python scripts/c3_time.py 2>&1 | grep "\[adapt\]" | tail -16
