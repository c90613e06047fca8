"""CPU oracle for parity tests — TEST INFRASTRUCTURE ONLY (see gpir_oracle.py)."""
