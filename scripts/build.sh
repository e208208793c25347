#!/bin/bash
# quiet in-tree build: prints errors only, exit code of make
make -s -j16 -C "$(dirname "$0")/../paper_0909_4969_b200" > /tmp/mb_build.log 2>&1
rc=$?
grep -E "error|Error" -A4 /tmp/mb_build.log | head -40
echo "build rc=$rc"
exit $rc
