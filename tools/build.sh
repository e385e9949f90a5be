#!/bin/bash
# developer helper: rebuild the product library, fail loudly
make -s -j8 -C $(dirname $0)/../paper_2508_01506_b200/csrc > /tmp/make.log 2>&1
rc=$?
grep -E "error|warning" /tmp/make.log | head -20
ls -la --time-style=+%H:%M:%S $(dirname $0)/../paper_2508_01506_b200/lib/libfsvd_b200.so
exit $rc
