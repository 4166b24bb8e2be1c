"""CPU ORACLE package — test infrastructure only (see ptrom_oracle.hpp header)."""
