#!/bin/bash
# round 2: A/B of two-rows-per-thread interior (248x8x2r) and x walls inside the interior tiles (XFUSE) at HEAD
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o_build.log 2>&1
for cfg in "" "WAVE25_INNER_TILE=248x8x2r" "WAVE25_XFUSE=1" "WAVE25_XFUSE=1 WAVE25_NO_ORIGIN=1" "WAVE25_INNER_TILE=null248x8x2" ; do
  echo "== $cfg" >> gpurun_out/qt_o.txt
  env $cfg timeout 300 python scripts/quick_time.py C3 stream 200 >> gpurun_out/qt_o.txt 2>&1
  env $cfg timeout 300 python scripts/prof_kinds.py C3 stream 10 >> gpurun_out/qt_o.txt 2>&1
done
echo "== C2 248x8x2r" >> gpurun_out/qt_o.txt
WAVE25_INNER_TILE=248x8x2r timeout 300 python scripts/quick_time.py C2 stream 400 >> gpurun_out/qt_o.txt 2>&1
timeout 600 python bench.py --precision fp64 --no-cpu-baseline --no-probe > gpurun_out/o_bench_fp64.json 2> gpurun_out/o_bench_fp64.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "variants and (248x8x2r or SEAM)" > gpurun_out/t_o.log 2>&1
echo "rc=$?" >> gpurun_out/t_o.log
echo done
