#!/bin/bash
# same-box A/B: old library build vs new (and BF_OPTS variants of the new), C2 timeline plain timings
cd "$(dirname "$0")/.."
OLD=${OLD:-tools/ab/lib_old.so}
for r in 1 2; do
  BF_LIB_PATH=$OLD timeout 300 python tools/timeline.py 32768 | grep opts | sed "s/^/old /"
  timeout 300 python tools/timeline.py 32768 | grep opts | sed "s/^/new /"
  for o in $NEWOPTS; do BF_OPTS=$o timeout 300 python tools/timeline.py 32768 | grep opts | sed "s/^/new /"; done
done
