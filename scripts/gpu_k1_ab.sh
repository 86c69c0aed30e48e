# K1 A/B: the in-tree build vs scripts/ab/tdkv_collect_<variant>.cu (run under gpurun;
# scripts/ab/ is git-ignored scratch; VARIANTS="a b" names scripts/ab/tdkv_collect_<name>.cu files)
set -e
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p /tmp/ab_build
for g in ${VARIANTS:-v1}; do
  mkdir -p /tmp/ab_build/$g
  cp paper_2604_03143_b200/csrc/*.cu paper_2604_03143_b200/csrc/*.cuh /tmp/ab_build/$g/
  cp scripts/ab/tdkv_collect_$g.cu /tmp/ab_build/$g/tdkv_collect.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include /tmp/ab_build/$g/*.cu -o /tmp/ab_build/libtdkv_$g.so
done
for lib in default ${VARIANTS:-v1} default ${VARIANTS:-v1}; do
  for c in c2 c3 c4 c1; do
    if [ $lib = default ]; then L=""; else L=/tmp/ab_build/libtdkv_$lib.so; fi
    TDKV_LIBRARY=$L python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-codec 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', d['value'], d['roofline']['frac'])"
  done
done
