#!/bin/bash
# A/B kernel experiments: build variant libraries in which some kernel sources
# come from an older commit (or from tools/variants_src/<name>/):
#   tools/build_variants.sh name:file@commit[,file@commit...] ...
# -> tools/variants/<name>/lib/libswattn_b200.so  (load with SWATTN_B200_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for spec in "$@"; do
  name=${spec%%:*}; files=${spec#*:}
  d=$ROOT/tools/variants/$name
  rm -rf $d; mkdir -p $d/lib/csrc $d/include
  cp $ROOT/paper_2509_24663_b200/csrc/*.cu $ROOT/paper_2509_24663_b200/csrc/*.cuh $ROOT/paper_2509_24663_b200/csrc/Makefile $d/lib/csrc/
  cp $ROOT/include/*.h $d/include/
  if [ "$files" != "$spec" ] && [ -n "$files" ]; then
    IFS=, read -ra FS <<< "$files"
    for f in "${FS[@]}"; do
      git -C $ROOT show ${f#*@}:paper_2509_24663_b200/csrc/${f%@*} > $d/lib/csrc/${f%@*}
    done
  fi
  if [ -d $ROOT/tools/variants_src/$name ]; then cp $ROOT/tools/variants_src/$name/* $d/lib/csrc/; fi
  make -s -C $d/lib/csrc -j8 EXTRA="$EXTRA" > $d/build.log 2>&1 || { tail -20 $d/build.log; exit 1; }
  echo "built $d/lib/libswattn_b200.so"
done
