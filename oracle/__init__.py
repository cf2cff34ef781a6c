"""TEST INFRASTRUCTURE ONLY: CPU checkers (see oracle/qcsim_oracle.c)."""
