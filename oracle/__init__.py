"""CPU oracle package (test infrastructure only; see oracle/bolt_oracle.c header)."""
