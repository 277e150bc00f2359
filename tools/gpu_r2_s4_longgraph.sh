# fourth-session A/B: split plans replay a graph of 4 pairs of steps (lib G) instead of one pair (lib A)
for rep in 1 2 3; do for L in G H; do
  python tools/time_shape.py 8 4 330 801 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c1 lib$L #"
  python tools/time_shape.py 10 5 2002 401 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2 lib$L #"
  python tools/time_shape.py 10 5 4004 401 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2b lib$L #"
  python tools/time_shape.py 9 4 700 801 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#n9 lib$L #"
done; done
