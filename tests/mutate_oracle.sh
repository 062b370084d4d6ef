#!/bin/bash
# Mutation check of the oracle pins: apply one sed edit to a scratch copy of
# oracle/nf_oracle.c and run tests/test_oracle.py; a surviving mutant = a missing pin.
# usage: (cd /tmp/mut && tests/mutate_oracle.sh "s/.../.../")
rm -rf r && mkdir r && cp -r /root/repo/oracle /root/repo/synth /root/repo/tests r/ && rm -f r/oracle/*.so
sed -i "$1" r/oracle/nf_oracle.c
if diff -q r/oracle/nf_oracle.c /root/repo/oracle/nf_oracle.c >/dev/null; then echo "NO-OP MUTATION: $1"; exit; fi
cd r && timeout 300 python -m pytest tests/test_oracle.py -q -x 2>&1 | tail -1 | sed "s|^|[$1] |"
