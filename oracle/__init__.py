"""ORACLE package -- test infrastructure only (see legpcg_port.py header)."""
