#!/bin/bash
# build compile-time variants of the engine into _ab/<name>/ (run on the dev box; the
# built copies travel to the GPU box with gpurun):  make_ab.sh name "-DFOO=1 -DBAR=2" ...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  d=_ab/$name; rm -rf $d; mkdir -p $d
  cp -r paper_2507_11289_b200 $d/; rm -rf $d/paper_2507_11289_b200/_build $d/paper_2507_11289_b200/libdsea.so
  mkdir -p $d/include && cp include/*.h $d/include/
  (cd $d && DSEA_NVCC_EXTRA="$defs" python -m paper_2507_11289_b200.build --force --verbose > build.log 2>&1) || { echo "build $name failed"; tail $d/build.log; }
  grep -A3 "k_force_tileILb0" $d/build.log | grep -o "Used [0-9]* registers" | head -1 | sed "s/^/$name: /"
done
