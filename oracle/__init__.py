"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/sa_oracle.c)."""
