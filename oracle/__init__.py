"""Test-infrastructure oracle for the STL hot path (see stl_oracle.py header)."""
