"""ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/meft_oracle.h). Never imported by the product path."""
