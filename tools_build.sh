#!/bin/bash
# developer helper: rebuild the product library, fail loudly
make -s -j8 -C /root/repo/paper_2508_01506_b200/csrc > /tmp/make.log 2>&1
rc=$?
grep -E "error|warning" /tmp/make.log | head -20
ls -la --time-style=+%H:%M:%S /root/repo/paper_2508_01506_b200/lib/libfsvd_b200.so
exit $rc
