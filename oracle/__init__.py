"""CPU oracle of the PreFT hot path — TEST INFRASTRUCTURE ONLY (see preft_oracle.py)."""
