#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family (tools/sanitize.py)
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
for t in memcheck racecheck synccheck; do
  echo "## $t" >> $OUT/sanitizers.txt
  timeout 900 compute-sanitizer --tool $t python tools/sanitize.py >> $OUT/sanitizers.txt 2>&1
done
grep -E "SUMMARY|^## " $OUT/sanitizers.txt
