# L=8 build+solve through several library builds (developer A/B); u compared bitwise with the first
first=""
for lib in "$@"; do
  timeout 300 python tools/solve_ab.py $lib /tmp/u_$(basename $lib).npy
  if [ -z "$first" ]; then first=/tmp/u_$(basename $lib).npy; else python -c "import numpy as np,sys; a=np.load('$first'); b=np.load('/tmp/u_$(basename $lib).npy'); print('bitwise vs first:', np.array_equal(a,b))"; fi
done
