#!/bin/bash
for W in 18432 18992 24576 36864 37984 12288 6144; do python scripts/narrow_rows.py 65536 $W; done
