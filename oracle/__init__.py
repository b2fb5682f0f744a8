"""CPU oracle (test infrastructure only). See oracle/sg_oracle.c header."""
