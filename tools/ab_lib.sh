#!/bin/bash
# A/B a command against an alternative build of the library: ab_lib.sh ALT_SO CMD...
# (runs CMD with the in-tree library, then with ALT_SO swapped in, then restores it)
alt=$1; shift
lib=paper_1011_5964_b200/libtvdeblur_b200.so
echo "== in-tree"; "$@"
cp $lib /tmp/ab_cur.so; cp $alt $lib
echo "== alt $alt"; "$@"
cp /tmp/ab_cur.so $lib
