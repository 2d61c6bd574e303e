"""CPU oracle for the IntAttention path -- test infrastructure only (see oracle.py)."""
