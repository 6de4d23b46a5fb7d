#!/bin/bash
# A/B of two library builds on the same box: bash tools/ab_shapes.sh OTHER.so
for i in 1 2; do
  XG_TAG=new bash tools/shapes.sh
  XG_LIB_PATH=$(realpath $1) XG_TAG=old bash tools/shapes.sh
done
