#!/bin/bash
# Dev helper: refuse to ship to the GPU box when the library is older than any
# CUDA source (a failed build would otherwise run the stale library).
lib=paper_1510_01041_b200/_lib/liblmsb200.so
for f in paper_1510_01041_b200/csrc/*.cu paper_1510_01041_b200/csrc/*.cuh include/*.h; do
  if [ "$f" -nt "$lib" ]; then echo "STALE: $f is newer than $lib"; exit 1; fi
done
exec /usr/local/graft/bin/gpurun "$@"
