"""Test infrastructure: CPU oracle of the reference inference path (see oracle.py)."""
