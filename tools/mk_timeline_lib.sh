#!/bin/bash
# build an instrumented copy of libdsmpnn.so into tools/tl/ and restore the clean build
set -e
mkdir -p tools/tl
cd /root/repo
python tools/instr_bwd2.py on
python -m paper_2402_15106_b200.build >/dev/null
cp paper_2402_15106_b200/libdsmpnn.so tools/tl/libdsmpnn.so
python tools/instr_bwd2.py restore
python -m paper_2402_15106_b200.build >/dev/null
echo built
