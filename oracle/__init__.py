"""CPU oracle for parity tests (test infrastructure only; see krul_oracle.hpp)."""
