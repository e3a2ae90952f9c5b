python tools/diag_graph.py crbd
python tools/diag_graph.py geometric
