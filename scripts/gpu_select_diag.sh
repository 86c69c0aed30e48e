python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/select_bench.py
python scripts/select_bench.py 1 4096
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_kernel python scripts/select_bench.py 2>&1 | grep -E "gpu__time" | sort | uniq -c | sort -rn | head -2
