(cd abold && python ../tools/quick_perf.py 2>&1 | tail -17 | cut -c1-120 | sed 's/^/OLD /')
python tools/quick_perf.py 2>&1 | tail -17 | cut -c1-120 | sed 's/^/NEW /'
