"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/tmpc_oracle.cpp header)."""
