"""CPU float64 oracle — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header)."""
