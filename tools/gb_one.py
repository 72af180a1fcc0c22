import os, sys
sys.path.insert(0, os.getcwd())
exec(open('tools/groupbench.py').read().split('out = {}')[0])
st.apply(circuit(16, True), budget=100000, tile_bits=12)
