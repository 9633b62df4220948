#!/bin/bash
# Copy one evidence pass (tools/gpu_evidence_r02.sh TAG) from gpurun_out/
# into profiles/r02/ and regenerate the markdown summaries + SUMMARY.md.
TAG=${1:?tag}; IN=gpurun_out; OUT=profiles/r02
set -e
tail -n 1 $IN/bench_$TAG.json > $OUT/bench.json
tail -n 1 $IN/bench_ref_$TAG.json > $OUT/bench_reference.json
cp $IN/launches_$TAG.csv $OUT/launches.csv
python tools/ncu_summary.py --launches $IN/launches_$TAG.csv > $OUT/launches.md
for k in gstream attn comb dexp logits gemm fold; do
  [ -f $IN/prof_${k}_$TAG.ncu-rep ] && python tools/ncu_summary.py --rep $IN/prof_${k}_$TAG.ncu-rep > $OUT/ncu_$k.md
done
cp $IN/pytest_gpu_$TAG.log $OUT/pytest_gpu.txt
cp $IN/smoke_$TAG.log $OUT/smoke.txt
[ -f $IN/fold_$TAG.txt ] && cp $IN/fold_$TAG.txt $OUT/fold.txt
[ -f $IN/fp2_rate_$TAG.txt ] && cp $IN/fp2_rate_$TAG.txt $OUT/fp2_rate.txt
rm -f $OUT/sanitize_*.log
for f in $IN/sanitize_${TAG}_*.log; do cp $f $OUT/$(basename $f | sed "s/_${TAG}_/_r02_/"); done
python tools/make_summary_r02.py > /dev/null
echo collected $TAG
