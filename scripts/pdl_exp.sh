#!/bin/bash
# programmatic dependent launch on/off (graphs on/off) across problem sizes
for shape in "3 256 256 32" "3 256 256 64" "3 256 256 256" "3 512 512 64" "3 512 512 512" "2 1024 1024 1" "2 512 512 1"; do
  for g in ${GRAPHS:-1 0}; do
    for p in 0 1; do
      python scripts/measure_shape.py $shape 1 $p $g 2>&1 | tail -1
    done
  done
done
