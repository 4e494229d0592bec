#!/bin/bash
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.log 2>&1; tail -1 /tmp/t.log; grep -A40 "^____" /tmp/t.log | head -50
HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.log 2>&1; tail -1 /tmp/t.log; grep -A40 "^____" /tmp/t.log | head -50
